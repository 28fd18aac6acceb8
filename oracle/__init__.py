"""CPU oracle for the threshold-RHG edge generator (arXiv 1606.09481).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_1606_09481_b200`` never imports it.

This file is argument marshalling (ctypes + numpy) around ``rhg_oracle.c``;
every piece of the method's arithmetic lives in the C file, which cites the
paper passage each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rhg_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_f64p = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, -O2, OpenMP, libquadmath)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", _SRC, "-o", _LIB,
               "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.orc_philox_words.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _u32p]
        L.orc_alpha.restype = ctypes.c_double
        L.orc_alpha.argtypes = [ctypes.c_double]
        L.orc_kbar_formula.restype = ctypes.c_double
        L.orc_kbar_formula.argtypes = [ctypes.c_double] * 3
        L.orc_target_radius.restype = ctypes.c_int
        L.orc_target_radius.argtypes = [ctypes.c_double] * 3 + [_f64p]
        L.orc_boundaries.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_double, _f64p]
        L.orc_uniforms.argtypes = [_u32p, _f64p, _f64p]
        L.orc_radius_from_uniform.restype = ctypes.c_double
        L.orc_radius_from_uniform.argtypes = [ctypes.c_double] * 3
        L.orc_sample_points.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_uint64, _f64p, _f64p]
        L.orc_angle_between.restype = ctypes.c_double
        L.orc_angle_between.argtypes = [ctypes.c_double] * 2
        L.orc_S.restype = ctypes.c_double
        L.orc_S.argtypes = [ctypes.c_double] * 4
        L.orc_cosh_dist_literal_quad.restype = ctypes.c_double
        L.orc_cosh_dist_literal_quad.argtypes = [ctypes.c_double] * 4 + [_f64p]
        L.orc_is_edge.restype = ctypes.c_int
        L.orc_is_edge.argtypes = [ctypes.c_double] * 5 + [ctypes.POINTER(ctypes.c_int)]
        for f in (L.orc_brute_force, L.orc_sweep):
            f.restype = ctypes.c_int64
            f.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double, _u32p, ctypes.c_uint64,
                          _u32p, _u8p, ctypes.c_uint64, _u64p, _u64p]
        L.orc_sweep_count.restype = ctypes.c_int64
        L.orc_sweep_count.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double,
                                      ctypes.c_uint64, ctypes.c_uint64, _u64p]
        L.orc_window.restype = ctypes.c_double
        L.orc_window.argtypes = [ctypes.c_double] * 3
        L.orc_rows.restype = ctypes.c_int64
        L.orc_rows.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double, ctypes.c_uint64,
                               _u32p, _u64p, _u32p, ctypes.c_uint64, _u32p]
        L.orc_row_ties.restype = ctypes.c_int64
        L.orc_row_ties.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double, ctypes.c_uint32,
                                   _u32p, _u8p, ctypes.c_uint64]
        L.orc_angle_order.argtypes = [ctypes.c_uint64, _f64p, _u32p, _u32p]
        L.orc_sweep_count_ordered.restype = ctypes.c_int64
        L.orc_sweep_count_ordered.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double,
                                              _u32p, _u32p, ctypes.c_uint64, ctypes.c_uint64,
                                              _u64p]
        L.orc_sweep_csr.restype = ctypes.c_int64
        L.orc_sweep_csr.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double, _u64p, _u32p,
                                    ctypes.c_uint64, _u32p, _u8p, ctypes.c_uint64, _u64p, _u64p]
        L.orc_sweep_digest.restype = ctypes.c_int64
        L.orc_sweep_digest.argtypes = [ctypes.c_uint64, _f64p, _f64p, ctypes.c_double, _u64p,
                                       _u64p, _u32p, _u8p, ctypes.c_uint64, _u64p]
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_radius_from_C.restype = ctypes.c_double
        L.orc_radius_from_C.argtypes = [ctypes.c_double] * 2
        L.orc_movement_init.argtypes = [ctypes.c_uint64, ctypes.c_uint64] + [ctypes.c_double] * 4 + \
            [_f64p, _f64p]
        L.orc_rotate.restype = ctypes.c_double
        L.orc_rotate.argtypes = [ctypes.c_double] * 2
        L.orc_radial_step.argtypes = [ctypes.c_double] * 4 + [_f64p, _f64p]
        L.orc_move_points.argtypes = [ctypes.c_uint64, _f64p, _f64p, _f64p, _f64p, ctypes.c_double,
                                      ctypes.c_double]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------- RNG + params
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return out


def philox_words(seed: int, i0: int, count: int) -> np.ndarray:
    out = np.zeros(4 * count, dtype=np.uint32)
    lib().orc_philox_words(seed, i0, count, _p(out, _u32p))
    return out.reshape(count, 4)


def alpha(gamma: float) -> float:
    return lib().orc_alpha(gamma)


def kbar_formula(n: float, alpha_: float, R: float) -> float:
    return lib().orc_kbar_formula(float(n), alpha_, R)


def target_radius(n: float, kbar: float, alpha_: float) -> float:
    R = ctypes.c_double()
    st = lib().orc_target_radius(float(n), float(kbar), float(alpha_), ctypes.byref(R))
    if st != 0:
        raise ValueError(f"orc_target_radius failed with status {st}")
    return R.value


def boundaries(R: float, L: int, p: float = 0.9) -> np.ndarray:
    c = np.zeros(L + 1)
    lib().orc_boundaries(R, L, p, _p(c, _f64p))
    return c


def uniforms(words) -> tuple[float, float]:
    w = np.asarray(words, dtype=np.uint32)
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().orc_uniforms(_p(w, _u32p), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def radius_from_uniform(u: float, alpha_: float, R: float) -> float:
    return lib().orc_radius_from_uniform(u, alpha_, R)


def sample_points(n: int, alpha_: float, R: float, seed: int):
    th = np.empty(n)
    r = np.empty(n)
    lib().orc_sample_points(n, alpha_, R, seed, _p(th, _f64p), _p(r, _f64p))
    return th, r


# ---------------------------------------------------------------- predicate
def angle_between(t1: float, t2: float) -> float:
    return lib().orc_angle_between(t1, t2)


def S(t1, r1, t2, r2) -> float:
    return lib().orc_S(t1, r1, t2, r2)


def cosh_dist_literal_quad(t1, r1, t2, r2):
    e = ctypes.c_double()
    v = lib().orc_cosh_dist_literal_quad(t1, r1, t2, r2, ctypes.byref(e))
    return v, e.value


def is_edge(t1, r1, t2, r2, R) -> tuple[bool, bool]:
    tie = ctypes.c_int()
    e = lib().orc_is_edge(t1, r1, t2, r2, R, ctypes.byref(tie))
    return bool(e), bool(tie.value)


def window(r: float, c: float, R: float) -> float:
    return lib().orc_window(r, c, R)


# ---------------------------------------------------------------- edge sets
class EdgeSet:
    """Undirected edges (u < v) in lexicographic order + near-tie pairs."""

    def __init__(self, pairs, ties, tie_edge):
        self.pairs = pairs          # (m, 2) uint32
        self.ties = ties            # (t, 2) uint32, u < v
        self.tie_edge = tie_edge    # (t,) bool: the __float128 decision

    @property
    def m(self):
        return len(self.pairs)


def _edge_call(fn, theta, r, R, cap_hint):
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n = len(theta)
    cap = max(int(cap_hint), 16)
    tcap = 1 << 16
    while True:
        pairs = np.zeros((cap, 2), dtype=np.uint32)
        ties = np.zeros((tcap, 2), dtype=np.uint32)
        te = np.zeros(tcap, dtype=np.uint8)
        nt = ctypes.c_uint64()
        need = ctypes.c_uint64()
        m = fn(n, _p(theta, _f64p), _p(r, _f64p), R, _p(pairs, _u32p), cap, _p(ties, _u32p),
               _p(te, _u8p), tcap, ctypes.byref(nt), ctypes.byref(need))
        if m >= 0:
            return EdgeSet(pairs[:m].copy(), ties[: nt.value].copy(), te[: nt.value].astype(bool))
        cap = max(cap, int(need.value) + 16)
        tcap = max(tcap, int(nt.value) + 16)


def brute_force(theta, r, R, cap_hint=None) -> EdgeSet:
    n = len(theta)
    return _edge_call(lib().orc_brute_force, theta, r, R, cap_hint or 8 * n + 1024)


def sweep(theta, r, R, cap_hint=None) -> EdgeSet:
    n = len(theta)
    return _edge_call(lib().orc_sweep, theta, r, R, cap_hint or 8 * n + 1024)


def sweep_count(theta, r, R, id_lo, id_hi):
    """Edges found from vertices with id in [id_lo, id_hi) (count only), and the
    number of candidate tests."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    t = ctypes.c_uint64()
    m = lib().orc_sweep_count(len(theta), _p(theta, _f64p), _p(r, _f64p), R, id_lo, id_hi,
                              ctypes.byref(t))
    return int(m), int(t.value)


def angle_order(theta):
    """(order, pos): ids sorted by (theta, id) and the inverse (uint32)."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    n = len(theta)
    order = np.zeros(n, dtype=np.uint32)
    pos = np.zeros(n, dtype=np.uint32)
    lib().orc_angle_order(n, _p(theta, _f64p), _p(order, _u32p), _p(pos, _u32p))
    return order, pos


def sweep_count_ordered(theta, r, R, order, pos, id_lo, id_hi):
    """Count-only sweep of owners [id_lo, id_hi) on a given angular order:
    (edges, tests)."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    t = ctypes.c_uint64()
    m = lib().orc_sweep_count_ordered(len(theta), _p(theta, _f64p), _p(r, _f64p), R,
                                      _p(order, _u32p), _p(pos, _u32p), id_lo, id_hi,
                                      ctypes.byref(t))
    return int(m), int(t.value)


class CSR:
    """Oracle CSR: both directions, rows ascending; plus near-tie pairs."""

    def __init__(self, row_ptr, col, ties, tie_edge):
        self.row_ptr, self.col, self.ties, self.tie_edge = row_ptr, col, ties, tie_edge


def sweep_csr(theta, r, R, cap_hint=None) -> CSR:
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n = len(theta)
    cap = max(int(cap_hint or 16 * n + 1024), 16)
    tcap = 1 << 16
    while True:
        rp = np.zeros(n + 1, dtype=np.uint64)
        col = np.empty(cap, dtype=np.uint32)
        ties = np.zeros((tcap, 2), dtype=np.uint32)
        te = np.zeros(tcap, dtype=np.uint8)
        nt, need = ctypes.c_uint64(), ctypes.c_uint64()
        m = lib().orc_sweep_csr(n, _p(theta, _f64p), _p(r, _f64p), R, _p(rp, _u64p),
                                _p(col, _u32p), cap, _p(ties, _u32p), _p(te, _u8p), tcap,
                                ctypes.byref(nt), ctypes.byref(need))
        if m >= 0:
            return CSR(rp, col[:m], ties[: nt.value].copy(), te[: nt.value].astype(bool))
        cap = max(cap, int(need.value) + 16)
        tcap = max(tcap, int(nt.value) + 16)
        del col


def sweep_digest(theta, r, R):
    """(m, deg[n] uint64, digest[n] uint64, ties, tie_edge): per-vertex degree and
    sum of mix64(neighbour) mod 2^64 of the sweep's edge set."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n = len(theta)
    tcap = 1 << 16
    while True:
        deg = np.zeros(n, dtype=np.uint64)
        dig = np.zeros(n, dtype=np.uint64)
        ties = np.zeros((tcap, 2), dtype=np.uint32)
        te = np.zeros(tcap, dtype=np.uint8)
        nt = ctypes.c_uint64()
        m = lib().orc_sweep_digest(n, _p(theta, _f64p), _p(r, _f64p), R, _p(deg, _u64p),
                                   _p(dig, _u64p), _p(ties, _u32p), _p(te, _u8p), tcap,
                                   ctypes.byref(nt))
        if nt.value <= tcap:
            return int(m), deg, dig, ties[: nt.value].copy(), te[: nt.value].astype(bool)
        tcap = int(nt.value) + 16


def mix64(w: int) -> int:
    return int(lib().orc_mix64(w))


def rows(theta, r, R, queries):
    """Brute-force neighbour lists (ascending ids) of the query vertices.
    Returns (offsets[nq+1], nbr, n_tie[nq])."""
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    q = np.ascontiguousarray(queries, dtype=np.uint32)
    nq = len(q)
    off = np.zeros(nq + 1, dtype=np.uint64)
    ntie = np.zeros(nq, dtype=np.uint32)
    cap = 1 << 20
    while True:
        nbr = np.zeros(cap, dtype=np.uint32)
        tot = lib().orc_rows(len(theta), _p(theta, _f64p), _p(r, _f64p), R, nq, _p(q, _u32p),
                             _p(off, _u64p), _p(nbr, _u32p), cap, _p(ntie, _u32p))
        if tot >= 0:
            return off, nbr[:tot].copy(), ntie
        cap = int(off[-1]) + 16


def row_ties(theta, r, R, v):
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    cap = 1024
    w = np.zeros(cap, dtype=np.uint32)
    e = np.zeros(cap, dtype=np.uint8)
    c = lib().orc_row_ties(len(theta), _p(theta, _f64p), _p(r, _f64p), R, v, _p(w, _u32p),
                           _p(e, _u8p), cap)
    c = min(c, cap)
    return w[:c].copy(), e[:c].astype(bool)


# ---------------------------------------------------------------- f2 / f1
def radius_from_C(n: float, C: float) -> float:
    """R = 2 ln n + C."""
    return lib().orc_radius_from_C(float(n), float(C))


def movement_init(n: int, seed: int, phi_range=(-1.0, 1.0), r_range=(-10.0, 1.0)):
    """Per-vertex step values (Appendix B ranges)."""
    tp = np.zeros(n, dtype=np.float64)
    tr = np.zeros(n, dtype=np.float64)
    lib().orc_movement_init(n, seed, phi_range[0], phi_range[1], r_range[0], r_range[1],
                            _p(tp, _f64p), _p(tr, _f64p))
    return tp, tr


def rotate(phi: float, tau_phi: float) -> float:
    return lib().orc_rotate(phi, tau_phi)


def radial_step(r: float, tau_r: float, R: float, alpha_: float):
    ro = ctypes.c_double()
    to = ctypes.c_double()
    lib().orc_radial_step(r, tau_r, R, alpha_, ctypes.byref(ro), ctypes.byref(to))
    return ro.value, to.value


def move_points(theta, r, tau_phi, tau_r, R: float, alpha_: float):
    """One movement step of every vertex (copies; tau_r returned with flipped signs)."""
    th = np.array(theta, dtype=np.float64)
    rr = np.array(r, dtype=np.float64)
    tp = np.ascontiguousarray(tau_phi, dtype=np.float64)
    tr = np.array(tau_r, dtype=np.float64)
    lib().orc_move_points(len(th), _p(th, _f64p), _p(rr, _f64p), _p(tp, _f64p), _p(tr, _f64p),
                          R, alpha_)
    return th, rr, tr


def num_threads() -> int:
    return lib().orc_num_threads()
