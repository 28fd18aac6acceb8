"""paper_1606_09481_b200 -- B200-native threshold random-hyperbolic-graph generator.

Thin ctypes binding over ``librhg.so`` (the C-ABI in ``include/rhg.h``).  This
module only marshals arguments: every step of the method (sampling, band
assignment, sorting, range queries, tests, emission) runs in the CUDA kernels of
``csrc/``.  PyTorch is used for device memory and streams only.

There is no CPU fallback: if the extension is missing, importing ``lib()`` raises.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RHG_LIB_PATH: an alternative build of the same library (experiments, scripts/);
# there is no other implementation behind it.
LIB_PATH = os.environ.get("RHG_LIB_PATH", os.path.join(_HERE, "librhg.so"))

RHG_OK, RHG_ERR_INVALID, RHG_ERR_CALIBRATION, RHG_ERR_WORKSPACE = 0, 2, 3, 4
RHG_ERR_CAPACITY, RHG_ERR_DOMAIN, RHG_ERR_CUDA = 5, 6, 7
RHG_CSR, RHG_EDGES_UNDIRECTED = 0, 1
FORMATS = {"csr": RHG_CSR, "edges": RHG_EDGES_UNDIRECTED, "pairs": RHG_EDGES_UNDIRECTED}

# Symbols include/rhg.h declares (tests check they are all exported).
ABI_SYMBOLS = ("rhg_target_radius", "rhg_band_boundaries", "rhg_workspace_bytes", "rhg_generate",
               "rhg_generate_with_radius", "rhg_generate_from_points", "rhg_sample_points",
               "rhg_philox_words", "rhg_status_string", "rhg_version", "rhg_last_cuda_error",
               "rhg_generate_with_C", "rhg_movement_init", "rhg_move_points",
               "rhg_stats_workspace_bytes", "rhg_graph_stats", "rhg_update_workspace_bytes",
               "rhg_update_moved")
STATS_BINS = 40


class RhgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rhg status {status}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("num_bands", ctypes.c_int), ("band_ratio", ctypes.c_double),
                ("heavy_threshold", ctypes.c_uint32), ("shard_index", ctypes.c_int),
                ("shard_count", ctypes.c_int), ("vertex_order", ctypes.c_int),
                ("wide_positions", ctypes.c_int), ("graph", ctypes.c_int)]


class Timing(ctypes.Structure):
    _fields_ = [("ms_sample", ctypes.c_float), ("ms_sort", ctypes.c_float),
                ("ms_index", ctypes.c_float), ("ms_count", ctypes.c_float),
                ("ms_scan", ctypes.c_float), ("ms_emit", ctypes.c_float),
                ("ms_copy", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("candidates", ctypes.c_uint64), ("certain", ctypes.c_uint64),
                ("launches", ctypes.c_uint64),
                ("emit_retested", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Stats(ctypes.Structure):
    _fields_ = [("num_edges", ctypes.c_uint64), ("max_degree", ctypes.c_uint64),
                ("mean_degree", ctypes.c_double), ("tail_count", ctypes.c_uint64),
                ("tail_exponent", ctypes.c_double), ("near_ties", ctypes.c_uint64),
                ("degree_hist", ctypes.c_uint64 * 40)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "degree_hist"}
        d["degree_hist"] = list(self.degree_hist)
        return d


class Update(ctypes.Structure):
    _fields_ = [("added", ctypes.c_void_p), ("removed", ctypes.c_void_p),
                ("capacity", ctypes.c_uint64), ("num_added", ctypes.POINTER(ctypes.c_uint64)),
                ("num_removed", ctypes.POINTER(ctypes.c_uint64)), ("row_capacity", ctypes.c_uint64),
                ("rows_needed", ctypes.POINTER(ctypes.c_uint64)), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("options", ctypes.c_void_p),
                ("timing", ctypes.c_void_p)]


class Output(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int), ("host_buffers", ctypes.c_int),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("pairs", ctypes.c_void_p),
                ("capacity_edges", ctypes.c_uint64), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("theta_out", ctypes.c_void_p),
                ("r_out", ctypes.c_void_p), ("num_edges", ctypes.POINTER(ctypes.c_uint64)),
                ("R_used", ctypes.POINTER(ctypes.c_double)),
                ("options", ctypes.POINTER(Options)), ("timing", ctypes.POINTER(Timing)),
                ("perm_out", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load the in-tree CUDA library; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        st = ctypes.c_int
        u64, f64, vp = ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.rhg_target_radius.restype = st
        L.rhg_target_radius.argtypes = [u64, f64, f64, ctypes.POINTER(f64)]
        L.rhg_band_boundaries.restype = st
        L.rhg_band_boundaries.argtypes = [u64, f64, ctypes.POINTER(Options),
                                          ctypes.POINTER(ctypes.c_int), ctypes.POINTER(f64)]
        L.rhg_workspace_bytes.restype = ctypes.c_size_t
        L.rhg_workspace_bytes.argtypes = [u64, ctypes.c_int, u64, ctypes.c_int,
                                          ctypes.POINTER(Options)]
        L.rhg_generate.restype = st
        L.rhg_generate.argtypes = [u64, f64, f64, u64, ctypes.POINTER(Output), vp]
        L.rhg_generate_with_radius.restype = st
        L.rhg_generate_with_radius.argtypes = [u64, f64, f64, u64, ctypes.POINTER(Output), vp]
        L.rhg_generate_from_points.restype = st
        L.rhg_generate_from_points.argtypes = [u64, vp, vp, f64, ctypes.POINTER(Output), vp]
        L.rhg_sample_points.restype = st
        L.rhg_sample_points.argtypes = [u64, f64, f64, u64, vp, vp, vp]
        L.rhg_philox_words.restype = st
        L.rhg_philox_words.argtypes = [u64, u64, u64, vp, vp]
        L.rhg_update_workspace_bytes.restype = ctypes.c_size_t
        L.rhg_update_workspace_bytes.argtypes = [u64, u64, u64, ctypes.POINTER(Options)]
        L.rhg_update_moved.restype = st
        L.rhg_update_moved.argtypes = [u64, vp, vp, f64, vp, u64, vp, vp, vp, vp,
                                       ctypes.POINTER(Update), vp]
        L.rhg_status_string.restype = ctypes.c_char_p
        L.rhg_status_string.argtypes = [ctypes.c_int]
        L.rhg_version.restype = ctypes.c_char_p
        L.rhg_version.argtypes = []
        L.rhg_generate_with_C.restype = st
        L.rhg_generate_with_C.argtypes = [u64, f64, f64, u64, ctypes.POINTER(Output), vp]
        L.rhg_movement_init.restype = st
        L.rhg_movement_init.argtypes = [u64, u64, f64, f64, f64, f64, vp, vp, vp]
        L.rhg_move_points.restype = st
        L.rhg_move_points.argtypes = [u64, vp, vp, vp, vp, f64, f64, vp]
        L.rhg_stats_workspace_bytes.restype = ctypes.c_size_t
        L.rhg_stats_workspace_bytes.argtypes = [u64]
        L.rhg_graph_stats.restype = st
        L.rhg_graph_stats.argtypes = [u64, ctypes.c_int, vp, vp, vp, u64, vp, vp, f64, f64, vp,
                                      ctypes.c_size_t, ctypes.POINTER(Stats), vp]
        L.rhg_last_cuda_error.restype = ctypes.c_char_p
        L.rhg_last_cuda_error.argtypes = []
        _lib = L
    return _lib


def _check(status: int):
    if status != RHG_OK:
        msg = lib().rhg_status_string(status).decode()
        if status == RHG_ERR_CUDA:
            msg += ": " + lib().rhg_last_cuda_error().decode()
        raise RhgError(status, msg)


def _torch():
    import torch
    return torch


def _stream_handle(stream=None):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


# --------------------------------------------------------------------------- host math
def target_radius(n: int, kbar: float, gamma: float) -> float:
    """getTargetRadius, computed by the library's host code."""
    R = ctypes.c_double()
    _check(lib().rhg_target_radius(n, kbar, gamma, ctypes.byref(R)))
    return R.value


def band_boundaries(n: int, R: float, num_bands: int = 0, band_ratio: float = 0.0) -> np.ndarray:
    o = Options(num_bands, band_ratio, 0)
    L = ctypes.c_int()
    c = (ctypes.c_double * 65)()
    _check(lib().rhg_band_boundaries(n, R, ctypes.byref(o), ctypes.byref(L), c))
    return np.array(c[: L.value + 1])


def workspace_bytes(n: int, fmt: str = "csr", capacity: int = 0, host_buffers: bool = False,
                    options=None) -> int:
    o = None if options is None else ctypes.byref(_options(options))
    return int(lib().rhg_workspace_bytes(n, FORMATS[fmt], capacity, int(host_buffers), o))


def _options(options) -> Options:
    if options is None:
        return Options(0, 0.0, 0, 0, 0)
    return Options(int(options.get("num_bands", 0)), float(options.get("band_ratio", 0.0)),
                   int(options.get("heavy_threshold", 0)), int(options.get("shard_index", 0)),
                   int(options.get("shard_count", 0)), int(options.get("vertex_order", 0)),
                   int(options.get("wide_positions", 0)), int(options.get("graph", 0)))


def version() -> str:
    return lib().rhg_version().decode()


# --------------------------------------------------------------------------- graphs
@dataclass
class Graph:
    n: int
    format: str
    R: float
    num_edges: int                 # directed entries (csr) or undirected edges (pairs)
    row_ptr: object = None         # torch int64 [n+1] (csr)
    col: object = None             # torch int32 (bits of uint32) [num_edges] (csr)
    pairs: object = None           # torch int32 [num_edges, 2] (pairs), u < v
    theta: object = None
    r: object = None
    timing: dict = field(default_factory=dict)
    perm: object = None            # vertex_order = 1: torch int32 [n], perm[id] = sample index

    @property
    def num_undirected(self) -> int:
        return self.num_edges // 2 if self.format == "csr" else self.num_edges


def _expected_capacity(n, kbar, fmt):
    if kbar is None:
        kbar = 16.0
    m_dir = n * kbar
    extra = 6.0 * math.sqrt(max(m_dir, 1.0)) + 0.15 * m_dir + 4096
    return int(m_dir + extra) if fmt == "csr" else int(m_dir / 2 + extra)


class Workspace:
    """Reusable device scratch for repeated calls (the bench keeps one)."""

    def __init__(self, device="cuda"):
        self.device = device
        self.buf = None

    def get(self, nbytes: int):
        torch = _torch()
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = None
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self.buf


def _run(call, n, fmt, kbar_hint, *, device, capacity, options, timing, workspace, stream,
         host_buffers, want_points, sample, out_bufs=None):
    torch = _torch()
    f = FORMATS[fmt]
    fmt = "csr" if f == RHG_CSR else "pairs"
    cap = int(capacity) if capacity is not None else _expected_capacity(n, kbar_hint, fmt)
    opts = _options(options)
    ws = workspace if workspace is not None else Workspace(device)
    for attempt in range(2):
        nbytes = int(lib().rhg_workspace_bytes(n, f, cap, int(host_buffers), ctypes.byref(opts)))
        wbuf = ws.get(nbytes)
        perm = None
        if out_bufs is not None:
            b = out_bufs(cap)
            row_ptr, col, pairs, theta, r = b[:5]
            perm = b[5] if len(b) > 5 else None
        else:
            kw = dict(device="cpu", pin_memory=True) if host_buffers else dict(device=device)
            row_ptr = torch.empty(n + 1, dtype=torch.int64, **kw) if f == RHG_CSR else None
            col = torch.empty(max(cap, 1), dtype=torch.int32, **kw) if f == RHG_CSR else None
            pairs = torch.empty((max(cap, 1), 2), dtype=torch.int32, **kw) if f != RHG_CSR else None
            theta = torch.empty(n, dtype=torch.float64, **kw) if (want_points and sample) else None
            r = torch.empty(n, dtype=torch.float64, **kw) if (want_points and sample) else None
        if opts.vertex_order == 1 and perm is None:
            kw = dict(device="cpu", pin_memory=True) if host_buffers else dict(device=device)
            perm = torch.empty(n, dtype=torch.int32, **kw)
        ne = ctypes.c_uint64()
        Ru = ctypes.c_double()
        tm = Timing()
        out = Output(f, int(host_buffers), _ptr(row_ptr), _ptr(col), _ptr(pairs), cap,
                     wbuf.data_ptr(), wbuf.numel(), _ptr(theta), _ptr(r), ctypes.pointer(ne),
                     ctypes.pointer(Ru), ctypes.pointer(opts),
                     ctypes.pointer(tm) if timing else None, _ptr(perm))
        st = call(ctypes.byref(out), _stream_handle(stream))
        if st == RHG_ERR_CAPACITY and capacity is None and attempt == 0:
            cap = int(ne.value)
            continue
        _check(st)
        m = int(ne.value)
        g = Graph(n=n, format=fmt, R=Ru.value, num_edges=m, theta=theta, r=r,
                  timing=tm.as_dict() if timing else {}, perm=perm)
        if f == RHG_CSR:
            g.row_ptr, g.col = row_ptr, col[:m]
        else:
            g.pairs = pairs[:m]
        return g
    raise RuntimeError("unreachable")


def generate(n: int, kbar: float, gamma: float, seed: int, fmt: str = "csr", *, device="cuda",
             capacity=None, options=None, timing=False, workspace=None, stream=None,
             host_buffers=False, return_points=False) -> Graph:
    """Algorithm 1 end to end on the GPU."""
    L = lib()
    return _run(lambda o, s: L.rhg_generate(n, kbar, gamma, seed, o, s), n, fmt, kbar,
                device=device, capacity=capacity, options=options, timing=timing,
                workspace=workspace, stream=stream, host_buffers=host_buffers,
                want_points=return_points, sample=True)


def generate_with_radius(n: int, R: float, alpha: float, seed: int, fmt: str = "csr", *,
                         device="cuda", capacity=None, options=None, timing=False, workspace=None,
                         stream=None, host_buffers=False, return_points=False,
                         kbar_hint=None) -> Graph:
    """Same with R given directly."""
    L = lib()
    return _run(lambda o, s: L.rhg_generate_with_radius(n, R, alpha, seed, o, s), n, fmt,
                kbar_hint, device=device, capacity=capacity, options=options, timing=timing,
                workspace=workspace, stream=stream, host_buffers=host_buffers,
                want_points=return_points, sample=True)


def generate_with_C(n: int, C: float, alpha: float, seed: int, fmt: str = "csr", *,
                    device="cuda", capacity=None, options=None, timing=False, workspace=None,
                    stream=None, host_buffers=False, return_points=False, kbar_hint=None) -> Graph:
    """R = 2 ln n + C."""
    L = lib()
    return _run(lambda o, s: L.rhg_generate_with_C(n, C, alpha, seed, o, s), n, fmt, kbar_hint,
                device=device, capacity=capacity, options=options, timing=timing,
                workspace=workspace, stream=stream, host_buffers=host_buffers,
                want_points=return_points, sample=True)


def movement_init(n: int, seed: int, phi_range=(-1.0, 1.0), r_range=(-10.0, 1.0), device="cuda",
                  stream=None):
    """Per-vertex step values of the dynamic model (Appendix B ranges)."""
    torch = _torch()
    tp = torch.empty(n, dtype=torch.float64, device=device)
    tr = torch.empty(n, dtype=torch.float64, device=device)
    _check(lib().rhg_movement_init(n, seed, phi_range[0], phi_range[1], r_range[0], r_range[1],
                                   tp.data_ptr(), tr.data_ptr(), _stream_handle(stream)))
    return tp, tr


def move_points(theta, r, tau_phi, tau_r, R: float, alpha: float, stream=None):
    """One movement step in place (rotation + Alg. 2 with reflection).
    All four are contiguous float64 CUDA tensors; tau_r changes sign on reflection."""
    for t in (theta, r, tau_phi, tau_r):
        assert t.is_cuda and t.dtype == _torch().float64 and t.is_contiguous()
    _check(lib().rhg_move_points(theta.numel(), theta.data_ptr(), r.data_ptr(), tau_phi.data_ptr(),
                                 tau_r.data_ptr(), R, alpha, _stream_handle(stream)))


def shard_offsets(counts) -> list:
    """Exclusive prefix of the per-shard edge counts: where shard s's edges start in
    the concatenation of all shards' outputs."""
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out + [acc]


def distributed_generate(n: int, kbar: float, gamma: float, seed: int, fmt: str = "csr", *,
                         group=None, device=None, **kw):
    """One graph sharded over the ranks of a torch.distributed group (one process per
    GPU): every rank samples and indexes all points, generates the edges it owns
    (shard = rank of world) and the ranks exchange one 8-byte edge count each
    (all_gather) for the global offsets.  Returns (graph shard, offsets, total)."""
    import torch.distributed as dist
    torch = _torch()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    opts = dict(kw.pop("options", None) or {})
    opts.update(shard_index=rank, shard_count=world)
    g = generate(n, kbar, gamma, seed, fmt, device=device or "cuda", options=opts, **kw)
    offsets, total = exchange_counts(g.num_edges, group=group)
    return g, offsets, total


def exchange_counts(num_edges: int, group=None):
    """all_gather of one uint64 edge count per rank -> (offsets, total)."""
    import torch.distributed as dist
    torch = _torch()
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    mine = torch.tensor([num_edges], dtype=torch.int64, device=dev)
    parts = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, mine, group=group)
    offs = shard_offsets([int(p.item()) for p in parts])
    return offs[:-1], offs[-1]


def graph_stats(g: "Graph", theta=None, r=None, k_min: float = 10.0, stream=None) -> dict:
    """On-device validation statistics (degree histogram, mean/max degree, tail MLE,
    near-tie edges) of a graph from this library.  theta/r: the
    points (CUDA, vertex-id order) for the near-tie count."""
    torch = _torch()
    L = lib()
    dev = g.row_ptr.device if g.format == "csr" else g.pairs.device
    ws = torch.empty(int(L.rhg_stats_workspace_bytes(g.n)), dtype=torch.uint8, device=dev)
    out = Stats()
    if g.format == "csr":
        args = (RHG_CSR, g.row_ptr.data_ptr(), g.col.data_ptr() if g.col.numel() else None, None, 0)
    else:
        args = (RHG_EDGES_UNDIRECTED, None, None, g.pairs.data_ptr() if g.num_edges else None,
                g.num_edges)
    _check(L.rhg_graph_stats(g.n, *args, _ptr(theta), _ptr(r), g.R, k_min, ws.data_ptr(),
                             ws.numel(), ctypes.byref(out), _stream_handle(stream)))
    d = out.as_dict()
    if theta is None:
        d["near_ties"] = None
    return d


def generate_from_points(theta, r, R: float, fmt: str = "csr", *, capacity=None, options=None,
                         timing=False, workspace=None, stream=None, kbar_hint=None) -> Graph:
    """Edges of a given point set (fp64 torch tensors; CUDA tensors, or CPU tensors
    for the host-buffer mode)."""
    torch = _torch()
    theta = theta.contiguous()
    r = r.contiguous()
    assert theta.dtype == torch.float64 and r.dtype == torch.float64 and theta.shape == r.shape
    n = theta.numel()
    host = not theta.is_cuda
    if host and not theta.is_pinned():
        theta, r = theta.pin_memory(), r.pin_memory()
    device = "cuda" if host else theta.device
    L = lib()
    hint = kbar_hint if kbar_hint is not None else 16.0
    return _run(lambda o, s: L.rhg_generate_from_points(n, theta.data_ptr(), r.data_ptr(), R, o, s),
                n, fmt, hint, device=device, capacity=capacity, options=options, timing=timing,
                workspace=workspace, stream=stream, host_buffers=host, want_points=False,
                sample=False)


@dataclass
class Delta:
    added: object      # torch int32 [num_added, 2], u < v
    removed: object    # torch int32 [num_removed, 2], u < v
    rows: int          # directed entries of the moved vertices' new rows
    timing: dict = field(default_factory=dict)


def update_moved(theta, r, R: float, moved, theta_old, r_old, old_row_ptr, old_col, *,
                 options=None, timing=False, workspace=None, stream=None, capacity=None,
                 row_capacity=None) -> Delta:
    """Edge delta of the dynamic model (rhg_update_moved): the new
    positions of all points, the moved vertex ids (int32, distinct) with their old
    positions, and the old graph's CSR (CUDA tensors).  Sizes its buffers from the
    library's required counts (one retry at most per buffer)."""
    torch = _torch()
    for t in (theta, r, theta_old, r_old):
        assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
    n, m = theta.numel(), moved.numel()
    dev = theta.device
    L = lib()
    opts = _options(options)
    old_deg = torch.diff(old_row_ptr)[moved.long()] if m else torch.zeros(1, device=dev)
    rcap = int(row_capacity) if row_capacity is not None else int(2 * old_deg.sum().item()) + 64 * m + 4096
    old_entries = int(old_row_ptr[-1].item())
    cap = int(capacity) if capacity is not None else rcap // 2 + 4096
    ws = workspace if workspace is not None else Workspace(dev)
    tm = Timing()
    for _ in range(3):
        wb = ws.get(int(L.rhg_update_workspace_bytes(n, rcap, old_entries, ctypes.byref(opts))))
        added = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev)
        removed = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev)
        na, nr, rn = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        u = Update(added.data_ptr(), removed.data_ptr(), cap, ctypes.pointer(na), ctypes.pointer(nr),
                   rcap, ctypes.pointer(rn), wb.data_ptr(), wb.numel(),
                   ctypes.cast(ctypes.pointer(opts), ctypes.c_void_p),
                   ctypes.cast(ctypes.pointer(tm), ctypes.c_void_p) if timing else None)
        st = L.rhg_update_moved(n, theta.data_ptr(), r.data_ptr(), R, moved.data_ptr() if m else None,
                                m, theta_old.data_ptr() if m else None,
                                r_old.data_ptr() if m else None, old_row_ptr.data_ptr(),
                                old_col.data_ptr() if old_col.numel() else None, ctypes.byref(u),
                                _stream_handle(stream))
        if st == RHG_ERR_WORKSPACE and rn.value > rcap:
            rcap = int(rn.value)
            continue
        if st == RHG_ERR_CAPACITY:
            cap = int(max(na.value, nr.value))
            continue
        _check(st)
        return Delta(added=added[: na.value], removed=removed[: nr.value], rows=int(rn.value),
                     timing=tm.as_dict() if timing else {})
    raise RuntimeError("rhg_update_moved: buffers could not be sized")


def sample_points(n: int, alpha: float, R: float, seed: int, device="cuda", stream=None):
    """K1 alone: the points rhg_generate_with_radius(n, R, alpha, seed) uses."""
    torch = _torch()
    th = torch.empty(n, dtype=torch.float64, device=device)
    r = torch.empty(n, dtype=torch.float64, device=device)
    _check(lib().rhg_sample_points(n, alpha, R, seed, th.data_ptr(), r.data_ptr(),
                                   _stream_handle(stream)))
    return th, r


def philox_words(seed: int, i0: int, count: int, device="cuda", stream=None):
    torch = _torch()
    out = torch.empty((count, 4), dtype=torch.int32, device=device)
    _check(lib().rhg_philox_words(seed, i0, count, out.data_ptr(), _stream_handle(stream)))
    return out


# --------------------------------------------------------------------------- helpers
def csr_to_pairs_numpy(row_ptr, col):
    """(u, v) with u < v from a symmetric CSR (host numpy)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    c = np.asarray(col).view(np.uint32).astype(np.int64)
    u = np.repeat(np.arange(len(rp) - 1, dtype=np.int64), np.diff(rp))
    keep = u < c
    p = np.stack([u[keep], c[keep]], axis=1).astype(np.uint32)
    key = p[:, 0].astype(np.uint64) << np.uint64(32) | p[:, 1].astype(np.uint64)
    return p[np.argsort(key, kind="stable")]
