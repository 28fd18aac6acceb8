#!/usr/bin/env python
"""Benchmark: threshold RHG generation (arXiv 1606.09481, Algorithm 1) on B200.

Default workload = BASELINE.json configs[2] ("config 3", the headline metric):
n = 1e7, kbar = 100, gamma = 3 (alpha = 1), Philox seed 3, CSR (uint64 row_ptr,
uint32 col).  One step = one rhg_generate call: sampling, band assignment, sort,
index, range queries with exact tests, count -> scan -> emit (every step of the
hot path, nothing cached).  Output buffers and workspace are preallocated.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Vertex ids: the timed steps use sample ids (rhg_options.vertex_order 0, the
SURVEY §8(a) contract); the same workload with ids in (slab, angle) order
(vertex_order 1, perm output) is timed beside it ("other_vertex_order"), and the
five BASELINE configs are reported at 1 GPU ("configs_1gpu", outside the timed loop).

Prints ONE JSON line (rank 0).  N > 1 (torchrun): by default ONE graph is sharded
over the ranks: every rank samples, sorts and indexes all points,
emits the rows of an equal share of the estimated work, and the ranks all_gather
one 8-byte edge count (NCCL) per step: strong scaling.  --mode replicas: every rank
generates its own independent graph (seed 3 + rank), weak scaling.
--impl reference times the CPU oracle (oracle/, C + OpenMP) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "undirected edges/sec at n=1e7,k̄=100,γ=3 (device-timed); HBM GB/s as % of peak"
CONFIG3 = dict(n=10_000_000, kbar=100.0, gamma=3.0, seed=3, fmt="csr")
WORKLOAD = "config3: threshold RHG n=1e7 kbar=100 gamma=3 seed=3, uint32 CSR (BASELINE.json configs[2])"


def peaks():
    p = {}
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    return p


# Measured FP64 pipe rate on this pool's B200 (profiles/r01_fp64_microbench.txt):
# DMUL 18.5e12/s, DFMA 17.0e12/s (~59-64 per clk per SM).  Used for the count pass,
# which is FP64-bound.
FP64_PEAK_OPS = 17.0e12
PROFILE_JSON = "r02_ncu_query_cfg3.json"  # committed ncu capture of the query kernels
FP64_OPS_PER_TEST = 13  # certified predicate: DADD, 2 DMUL + 3 DFMA (sin poly), 5 DMUL, DADD, DFMA


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.th = threading.Thread(target=rd, daemon=True)
        self.th.start()

    def wait_first(self, timeout=5.0):
        """Block until nvidia-smi printed its first row, so the sampling covers the
        timed region (the rows before it are dropped)."""
        t0 = time.time()
        while self.proc is not None and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.rows = []

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for nm, v in zip(names, r[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def reduce_over_ranks(tot_ms: float, edges: float, device, world: int):
    """Whole-job numbers: the slowest rank's timed-loop time (max) and the edges
    generated by all ranks (sum).  Replicas share no data; this is the only
    collective (timing bookkeeping, not the data path)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([tot_ms], dtype=torch.float64, device=device)
    e = torch.tensor([edges], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
    return float(t.item()), float(e.item())


def replica_seed(base_seed: int, rank: int) -> int:
    """Independent graph per rank (weak scaling): Philox key = base seed + rank."""
    return base_seed + rank


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


PAPER_CONTEXT = {
    "hardware": "2 x 8-core Intel Xeon E5-2680 @ 2.7 GHz, 256 GB, up to 32 threads (HT), "
                "C++11 + OpenMP in NetworKit, TBB malloc (PAPER.md:300-301)",
    "claim": "10 million vertices and 1G edges in under one minute (PAPER.md:12, 39); "
             "speedup 3-60 over the previous quadtree generator (PAPER.md:11, 314)",
    "edge_sampling_s": {"workload": "n=1e7, kbar=6, gamma=3 (~3e7 undirected edges)",
                        "1_thread": 47.20, "16_threads": round(47.20 / 13.48, 2),
                        "32_threads": round(47.20 / 18.38, 2),
                        "source": "PAPER.md:366-379 (Fig. 3 normaliser 47.20 s; speedups 13.48, 18.38)"},
    "runtime_fit": "T(n,m) = (7.07 n log10 n + 2.23 m + 891) 1e-8 s (PAPER.md:358): "
                   "16.1 s at n=1e7, m=5e8",
    "note": "context only: another machine, whole-generator numbers except edge_sampling_s",
}

ORACLE_C5_ROWS = 32  # config-5 sampled-degree check size in the bench (the GPU tests run 100)


def oracle_config(cfg: int, oracle):
    """The CPU oracle on BASELINE config `cfg`, on the box's host cores, with its
    steps timed separately: Philox sampling, the angular sort, and
    the sweep (brute force for config 1).  Config 5: the
    sampled-degree check (brute-force degrees of ORACLE_C5_ROWS seeded vertices over
    all 1e8 points), not a full graph.  Returns a dict (times in s)."""
    import numpy as np
    n, kbar, gamma, seed, _fmt = ALL_CONFIGS[cfg]
    a = oracle.alpha(gamma)
    R = oracle.target_radius(n, kbar, a)
    t0 = time.perf_counter()
    th, r = oracle.sample_points(n, a, R, seed)
    t1 = time.perf_counter()
    out = {"cores": oracle.num_threads(), "sample_s": t1 - t0}
    if cfg == 1:
        es = oracle.brute_force(th, r, R)
        t2 = time.perf_counter()
        out.update(kind="brute force, all n(n-1)/2 pairs", sort_s=0.0, sweep_s=t2 - t1,
                   undirected_edges=es.m, tests=n * (n - 1) // 2)
    elif cfg == 5:
        q = np.random.default_rng(5).choice(n, ORACLE_C5_ROWS, replace=False).astype(np.uint32)
        off, _nbr, _t = oracle.rows(th, r, R, q)
        t2 = time.perf_counter()
        out.update(kind=f"sampled-degree check: {len(q)} seeded vertices, brute force over all "
                        f"{n} points (count + fill passes)", sort_s=0.0, sweep_s=t2 - t1,
                   queries=q, degrees=np.diff(off.astype(np.int64)), tests=2 * len(q) * (n - 1))
        return out
    else:
        order, pos = oracle.angle_order(th)
        t2 = time.perf_counter()
        m, tests = oracle.sweep_count_ordered(th, r, R, order, pos, 0, n)
        t3 = time.perf_counter()
        out.update(kind="radius-ordered angular sweep (count), all vertices", sort_s=t2 - t1,
                   sweep_s=t3 - t2, undirected_edges=m, tests=tests)
    out["total_s"] = out["sample_s"] + out["sort_s"] + out["sweep_s"]
    out["edges_per_s"] = out["undirected_edges"] / out["total_s"]
    return out


def run_reference(args):
    """The oracle arm: config 3 on the CPU oracle, as it stands, on the host cores.
    Sampling and the angular sort run once (timed); the K timed steps each sweep
    1/K of the owners (ids [k n/K, (k+1) n/K)), so the K steps together are one
    full oracle run; each step is charged its sweep time plus 1/K of the sampling
    and sort time.  value = all edges / all charged time = the full oracle's rate
    (the same protocol as the cpu_baseline of the GPU arm's line)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    c = CONFIG3
    n = c["n"]
    a = oracle.alpha(c["gamma"])
    R = oracle.target_radius(n, c["kbar"], a)
    t0 = time.perf_counter()
    th, r = oracle.sample_points(n, a, R, c["seed"])
    t1 = time.perf_counter()
    order, pos = oracle.angle_order(th)
    t2 = time.perf_counter()
    fixed = t2 - t0
    for w in range(args.warmup):  # tiny slices: page in and warm the caches
        oracle.sweep_count_ordered(th, r, R, order, pos, w * 1000, (w + 1) * 1000)
    K = max(1, args.steps)
    ms, secs, tests = [], [], 0
    for k in range(K):
        lo, hi = k * n // K, (k + 1) * n // K
        s0 = time.perf_counter()
        m, t = oracle.sweep_count_ordered(th, r, R, order, pos, lo, hi)
        secs.append(time.perf_counter() - s0 + fixed / K)
        ms.append(m)
        tests += t
    value = sum(ms) / sum(secs)
    sample = (f"config 3 in full over the {K} steps: sampling {t1 - t0:.2f} s + angular sort "
              f"{t2 - t1:.2f} s once (charged 1/{K} per step), each step the count sweep of "
              f"1/{K} of the owners; {sum(ms)} undirected edges, {tests} tests")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox-sampled points, seed 3)",
            "config": {"workload": WORKLOAD, "n": n, "kbar": c["kbar"], "gamma": c["gamma"],
                       "format": "count only (the oracle's sweep decides every candidate pair)"},
            "cpu_baseline": {"value": value, "unit": "edges/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": sample, "cpu": cpu_model(),
                             "sample_s": t1 - t0, "sort_s": t2 - t1, "sweep_s": sum(secs) - fixed},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "paper_context": PAPER_CONTEXT}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1606_09481_b200 as rhg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL between GPUs; RHG_BENCH_BACKEND=gloo lets a test run ranks that share a GPU
        dist.init_process_group(os.environ.get("RHG_BENCH_BACKEND", "nccl"))
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    c = CONFIG3
    shard = args.mode == "shard" and world > 1
    # replicas: an independent graph per rank (weak scaling); shard: one graph, each
    # rank emits 1/N of it and the ranks all_gather one edge count (strong scaling)
    seed = c["seed"] if shard else replica_seed(c["seed"], rank)
    opts = dict(vertex_order=args.order, graph=0 if args.no_graph else 1)
    if shard:
        opts.update(shard_index=rank, shard_count=world)
    # a dedicated stream: CUDA-graph replay (rhg_options.graph) cannot capture the
    # legacy default stream
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ws = rhg.Workspace(dev)

    # warm-up: also sizes the output exactly (capacity protocol)
    g = rhg.generate(c["n"], c["kbar"], c["gamma"], seed, c["fmt"], device=dev, workspace=ws,
                     options=opts)
    cap = g.num_edges
    row_ptr = torch.empty(c["n"] + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    perm = torch.empty(c["n"], dtype=torch.int32, device=dev)
    del g
    bufs = lambda _cap: (row_ptr, col, None, None, None, perm)

    def step(timing=False, options=opts):
        g = rhg._run(lambda o, s: rhg.lib().rhg_generate(c["n"], c["kbar"], c["gamma"], seed, o, s),
                     c["n"], c["fmt"], c["kbar"], device=dev, capacity=cap, options=options,
                     timing=timing, workspace=ws, stream=stream, host_buffers=False,
                     want_points=False, sample=True, out_bufs=bufs)
        if shard:
            g.offsets, g.total = rhg.exchange_counts(g.num_edges)  # the 8-byte NCCL all_gather
        return g

    for _ in range(args.warmup):
        step()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    # the other vertex order, same protocol, fewer steps (reported beside the headline)
    other = dict(opts, vertex_order=1 - args.order)
    for _ in range(2):
        step(options=other)
    torch.cuda.synchronize()
    oth_ms = []
    for i in range(max(3, args.steps // 3)):
        flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        go = step(options=other)
        e1.record(stream)
        torch.cuda.synchronize()
        oth_ms.append(e0.elapsed_time(e1))
    other_line = {"vertex_order": other["vertex_order"],
                  "value": (go.num_edges / 2.0) / (statistics.median(oth_ms) * 1e-3),
                  "ms_per_step": statistics.median(oth_ms), "steps": len(oth_ms)}
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phases = []
    clk = ClockSampler(gpu)
    clk.start()
    clk.wait_first()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    last = None
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # L2 flush between timed steps, outside the events
        ev[i][0].record(stream)
        last = step()  # graph replay of the whole call (eager with --no-graph)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    # per-phase split: library events need eager launches, so a few more steps
    for i in range(5):
        flush.fill_(i & 0xFF)
        phases.append(step(timing=True).timing)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    red_dev = dev if world == 1 or dist.get_backend() == "nccl" else "cpu"
    tot_ms, m_und_total = reduce_over_ranks(tot_ms, last.num_edges / 2.0, red_dev, world)
    ms_per_step = tot_ms / args.steps  # m_und_total: undirected edges per step, all ranks
    value = m_und_total / (ms_per_step * 1e-3)

    # per-phase device times (events on this stream, inside the timed steps)
    keys = ["ms_sample", "ms_sort", "ms_index", "ms_count", "ms_scan", "ms_emit"]
    ph = {k: statistics.median([p[k] for p in phases]) for k in keys}
    cand = phases[-1]["candidates"]
    launches = int(phases[-1]["launches"]) * args.steps  # the same kernels every step
    n = c["n"]
    m_dir = last.num_edges
    P = peaks()
    hbm_peak = P.get("hbm_gbs", 6650.0)
    # Dominant phase: the emit pass (light k_query<EMIT> + hub k_heavy<EMIT>, joined on
    # the caller's stream; library-recorded CUDA events).  Algorithmic bytes: the CSR
    # col write (4 B) and the id gather (4 B) per directed edge, the row_ptr pair
    # (16 B) and the query record (32 B) per vertex.
    # vertex_order 1 writes ids without the gather: 4 B per directed edge, plus the row
    # offset (8 B), the certain count (4 B) and the query record (32 B) per vertex.
    emit_bytes = (4 * m_dir + 44 * n) if args.order == 1 else (8 * m_dir + 16 * n + 32 * n)
    count_ops = FP64_OPS_PER_TEST * cand
    count_s, emit_s = ph["ms_count"] * 1e-3, ph["ms_emit"] * 1e-3
    traffic = None
    try:  # ncu dram bytes of the same kernel, committed capture (profiles/)
        prof = json.load(open(os.path.join(ROOT, "profiles", PROFILE_JSON)))
        kq = prof["kernels"]["k_query<EMIT,seq>" if args.order == 1 else "k_query<EMIT>"]
        traffic = (kq["dram_read_GB"] + kq["dram_write_GB"]) * 1e9
    except Exception:
        pass
    roof_emit = {"kernel": "emit phase: k_query<EMIT> + k_heavy<EMIT>", "bound": "hbm",
                 "achieved": emit_bytes / emit_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                 "frac": emit_bytes / emit_s / 1e9 / hbm_peak, "traffic": traffic,
                 "algorithmic_bytes": emit_bytes,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                 "traffic_source": f"profiles/{PROFILE_JSON} (ncu dram__bytes_read+write, "
                                   "light emit kernel, one launch)"}
    roof_count = {"kernel": "count phase: k_query<COUNT> + k_heavy<COUNT>", "bound": "alu",
                  "achieved": count_ops / count_s / 1e12, "peak": FP64_PEAK_OPS / 1e12,
                  "unit": "TFLOP/s (fp64 ops)", "frac": count_ops / count_s / FP64_PEAK_OPS,
                  "traffic": None,
                  "peak_source": "measured DFMA rate, profiles/r01_fp64_microbench.txt",
                  "note": "issue-bound (ncu IPC ~3.0 of 4), not FP64-pipe bound"}
    dominant = roof_emit if emit_s >= count_s else roof_count
    # what actually bounds the two query kernels: the instruction issue rate
    # (148 SMs x 4 schedulers x the SM clock), from the committed ncu capture
    issue = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", PROFILE_JSON)))
        clk = 1.965e9
        peak = 148 * 4 * clk
        issue = {"peak_warp_inst_per_s": peak, "source": f"profiles/{PROFILE_JSON}"}
        for lab in ("k_query<COUNT>", "k_query<EMIT,seq>" if args.order == 1 else "k_query<EMIT>"):
            k = prof["kernels"][lab]
            rate = k["inst_executed"] / (k["duration_ms"] * 1e-3)
            issue[lab] = {"warp_inst": k["inst_executed"], "ms": k["duration_ms"],
                          "achieved": rate, "frac": rate / peak,
                          "fp64_pipe_pct": k.get("fp64_pipe_pct"),
                          "active_threads_per_inst": k.get("threads_per_inst"),
                          "branch_targets_uniform_pct": k.get("branch_targets_uniform_pct"),
                          "l2_hit_pct": k.get("l2_hit_pct"),
                          "top_stalls_per_issue": k.get("top_stalls_per_issue")}
    except Exception:
        pass
    # north-star convention: points read (32 B) + 8 B per emitted directed edge, over query+emit
    ns_bytes = 32 * n + 8 * m_dir
    qe_s = count_s + ph["ms_scan"] * 1e-3 + emit_s
    north_star = {"query_emit_ms": qe_s * 1e3, "bytes": ns_bytes,
                  "GBps": ns_bytes / qe_s / 1e9, "frac_of_measured": ns_bytes / qe_s / 1e9 / hbm_peak,
                  "frac_of_8TBps": ns_bytes / qe_s / 1e9 / 8000.0}

    e2e = None
    cpu = None
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = five_configs(rhg, torch, dev, flush, args.order, hbm_peak, 0 if args.no_graph else 1)
    if rank == 0 and world == 1 and not args.no_e2e:
        e2e = measure_e2e(rhg, torch, c, seed, dev, ws, cap, args, opts)
        e2e["from_points"] = measure_e2e_points(rhg, torch, c, seed, dev, ws, cap, args, opts)
    near = None
    dyn = None
    if rank == 0 and world == 1:
        near = near_tie_stats(rhg, torch, c, seed, dev, opts)
        if not args.no_dynamic:
            dyn = dynamic_update(rhg, torch, c, seed, dev)
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        o3 = oracle_config(3, oracle)
        cpu = {"value": o3["edges_per_s"], "unit": "edges/s", "cores": o3["cores"],
               "kind": "oracle",
               "sample": (f"config 3 in full (not a sample): Philox sampling {o3['sample_s']:.2f} s"
                          f" + angular sort {o3['sort_s']:.2f} s + count sweep over all "
                          f"{n} owners {o3['sweep_s']:.2f} s; {o3['undirected_edges']} undirected "
                          f"edges, {o3['tests']} tests; value = edges / (sum of the three)"),
               "cpu": cpu_model(), "sample_s": o3["sample_s"], "sort_s": o3["sort_s"],
               "sweep_s": o3["sweep_s"], "edges_match_gpu": o3["undirected_edges"] == m_dir // 2}
        if configs is not None:
            add_oracle_to_configs(configs, oracle, o3)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "strong" if shard else "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (Philox4x32-10-sampled points, seed 3 + rank)",
                "config": {"workload": WORKLOAD, "n": n, "kbar": c["kbar"], "gamma": c["gamma"],
                           "format": "csr",
                           "vertex_order": (f"{args.order}: " + ("ids in (slab, angle) order, "
                                            "perm[id] = sample index also output" if args.order == 1
                                            else "ids = sample index")),
                           "parallelism": ("shards" if shard else "replicas") if world > 1 else "single",
                           "l2": "flushed between steps (256 MiB fill outside the step events)",
                           "launch": ("eager" if args.no_graph else
                                      "CUDA-graph replay of each call (rhg_options.graph)"),
                           "undirected_edges_per_step_per_rank": m_dir // 2},
                "roofline": dominant, "roofline_other": roof_emit if dominant is roof_count else roof_count,
                "north_star_hbm": north_star, "issue_rate": issue,
                "phases_ms": ph, "candidates": cand, "other_vertex_order": other_line,
                "configs_1gpu": configs, "near_ties": near, "dynamic_update": dyn,
                "cpu_baseline": cpu, "paper_context": PAPER_CONTEXT, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "wall_s_timed_loop": wall,
                "library": rhg.version()}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


ALL_CONFIGS = {1: (10_000, 6.0, 3.0, 1, "csr"), 2: (1_000_000, 10.0, 3.0, 2, "csr"),
               3: (10_000_000, 100.0, 3.0, 3, "csr"), 4: (1_000_000, 32.0, 2.2, 4, "csr"),
               5: (100_000_000, 16.0, 2.7, 5, "pairs")}


def five_configs(rhg, torch, dev, flush, order, hbm_peak, graph, steps=5):
    """The north star's per-config report at 1 GPU (BASELINE.json configs 1-5):
    edges/s and generation time (device events around rhg_generate, L2 flushed
    between steps), and the north-star HBM fraction (32 B/pt + 8 B per directed edge
    over the query+scan+emit phases)."""
    out = {}
    stream = torch.cuda.current_stream()
    for cfg, (n, kbar, gamma, seed, fmt) in ALL_CONFIGS.items():
        ws = rhg.Workspace(dev)
        opts = dict(vertex_order=order, graph=graph)
        g = rhg.generate(n, kbar, gamma, seed, fmt, device=dev, workspace=ws, options=opts)
        cap = g.num_edges
        del g
        rp = torch.empty(n + 1, dtype=torch.int64, device=dev) if fmt == "csr" else None
        col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev) if fmt == "csr" else None
        pr = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev) if fmt != "csr" else None
        perm = torch.empty(n, dtype=torch.int32, device=dev)

        def call(timing):
            return rhg._run(lambda o, s: rhg.lib().rhg_generate(n, kbar, gamma, seed, o, s),
                            n, fmt, kbar, device=dev, capacity=cap, options=opts, timing=timing,
                            workspace=ws, stream=stream, host_buffers=False, want_points=False,
                            sample=True, out_bufs=lambda _c: (rp, col, pr, None, None, perm))
        ms, qe = [], []
        for i in range(steps + 2):
            flush.fill_(i & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g = call(False)
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                ms.append(e0.elapsed_time(e1))
        for i in range(3):
            flush.fill_(i & 0xFF)
            t = call(True).timing
            qe.append(t["ms_count"] + t["ms_scan"] + t["ms_emit"])
        und = g.num_edges // 2 if fmt == "csr" else g.num_edges
        if cfg == 5:  # degrees of the oracle's sampled vertices (config-5 check)
            import numpy as np
            q = np.random.default_rng(5).choice(n, ORACLE_C5_ROWS, replace=False)
            P = g.pairs.to(torch.int64) & 0xFFFFFFFF
            qd = torch.from_numpy(q.astype(np.int64)).to(dev)
            gpu_c5_deg = [int((P[:, 0] == v).sum() + (P[:, 1] == v).sum()) for v in qd]
            del P
        m_dir = 2 * und
        t_ms, q_ms = statistics.median(ms), statistics.median(qe)
        nb = 32 * n + 8 * m_dir
        out[str(cfg)] = {"n": n, "kbar": kbar, "gamma": gamma, "seed": seed, "format": fmt,
                         "undirected_edges": und, "ms_per_generation": t_ms,
                         "edges_per_s": und / (t_ms * 1e-3), "query_emit_ms": q_ms,
                         "hbm_frac_north_star": nb / (q_ms * 1e-3) / 1e9 / hbm_peak,
                         "steps": len(ms)}
        if cfg == 5:
            out[str(cfg)]["gpu_sampled_degrees"] = gpu_c5_deg
        del g, ws, rp, col, pr, perm
        torch.cuda.empty_cache()
    return out


def add_oracle_to_configs(configs, oracle, o3):
    """Attach the CPU oracle's time to each config of configs_1gpu (same run, host
    cores): full oracle for configs 1-4, the sampled-degree check for config 5."""
    for cfg in (1, 2, 3, 4, 5):
        o = o3 if cfg == 3 else oracle_config(cfg, oracle)
        e = configs[str(cfg)]
        d = {"cores": o["cores"], "kind": o["kind"], "sample_s": round(o["sample_s"], 3),
             "sort_s": round(o["sort_s"], 3), "sweep_s": round(o["sweep_s"], 3),
             "tests": o["tests"]}
        if cfg == 5:
            gd = e.pop("gpu_sampled_degrees", None)
            d["vertices"] = len(o["queries"])
            d["degrees_match_gpu"] = (gd == o["degrees"].tolist()) if gd is not None else None
            d["note"] = ("oracle on its own points, GPU on its own sampled points (r within "
                         "8 ulp): equal unless a near tie (GPU tests compare on identical points)")
        else:
            d.update(total_s=round(o["total_s"], 3), edges_per_s=o["edges_per_s"],
                     undirected_edges=o["undirected_edges"],
                     edges_match_gpu=o["undirected_edges"] == e["undirected_edges"],
                     gpu_speedup_vs_oracle=o["total_s"] / (e["ms_per_generation"] * 1e-3))
        e["oracle"] = d


def near_tie_stats(rhg, torch, c, seed, dev, opts):
    """North star: GPU edges inside the 1e-12 cosh R window, counted on the device
    (rhg_graph_stats) for the headline graph, outside the timed
    region.  The oracle-side comparison is in tests/test_gpu_fullsize.py."""
    g = rhg.generate(c["n"], c["kbar"], c["gamma"], seed, c["fmt"], device=dev,
                     options=dict(opts, graph=0), return_points=True)
    st = rhg.graph_stats(g, g.theta, g.r, k_min=2 * c["kbar"])
    out = {"edges_in_window": st["near_ties"], "window": "|cosh d - cosh R| <= 1e-12 cosh R",
           "mean_degree": st["mean_degree"], "tail_exponent_mle_k>=2kbar": st["tail_exponent"],
           "max_degree": st["max_degree"],
           "parity_log": "profiles/r02_near_ties.jsonl (full edge sets vs the oracle)"}
    del g
    torch.cuda.empty_cache()
    return out


def dynamic_update(rhg, torch, c, seed, dev, fracs=(0.01, 0.05, 0.12), reps=3):
    """SURVEY §8(f) f1 / PAPER.md:387-389: updating the config-3 graph after a
    fraction of the vertices moved (one step of the dynamic model, rotation + Alg. 2
    with the Appendix B step ranges) against generating the graph of the new
    positions from scratch (rhg_generate_from_points).  Device times (CUDA events),
    median of `reps`, outside the headline's timed loop."""
    n = c["n"]
    a = (c["gamma"] - 1.0) / 2.0
    R = rhg.target_radius(n, c["kbar"], c["gamma"])
    th, r = rhg.sample_points(n, a, R, seed, device=dev)
    g0 = rhg.generate_from_points(th, r, R, "csr")
    tp, tr = rhg.movement_init(n, seed + 100, device=dev)
    th1, r1 = th.clone(), r.clone()
    rhg.move_points(th1, r1, tp, tr, R, a)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    perm = torch.randperm(n, device=dev, generator=gen)
    stream = torch.cuda.current_stream()
    ws_u, ws_g = rhg.Workspace(dev), rhg.Workspace(dev)
    out = {"workload": "config 3 graph (CSR), a random subset of the vertices moved by one "
                       "step of the dynamic model", "rows": {}}

    def timed(fn):
        ms = []
        res = None
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.median(ms[1:]), res

    for f in fracs:
        ids = torch.sort(perm[: int(f * n)]).values
        th_n, r_n = th.clone(), r.clone()
        th_n[ids], r_n[ids] = th1[ids], r1[ids]
        idx32 = ids.to(torch.int32)
        tho, ro = th[ids].contiguous(), r[ids].contiguous()
        t_u, d = timed(lambda: rhg.update_moved(th_n, r_n, R, idx32, tho, ro, g0.row_ptr, g0.col,
                                                workspace=ws_u))
        t_g, g1 = timed(lambda: rhg.generate_from_points(th_n, r_n, R, "csr", workspace=ws_g,
                                                          kbar_hint=c["kbar"]))
        out["rows"][f"{f:.0%}"] = {"moved": int(ids.numel()), "update_ms": t_u,
                                   "full_generation_ms": t_g, "speedup": t_g / t_u,
                                   "removed": int(d.removed.shape[0]), "added": int(d.added.shape[0]),
                                   "edges_after": g1.num_edges // 2}
        del g1, d, th_n, r_n
        torch.cuda.empty_cache()
    del g0
    torch.cuda.empty_cache()
    return out


def measure_e2e_points(rhg, torch, c, seed, dev, ws, cap, args, opts):
    """The C-ABI call that carries input payload: rhg_generate_from_points with the
    n points (theta, r: 16 B each) in page-locked HOST memory and the CSR written to
    page-locked host buffers; both copies are inside the timed region (the library
    stages them through the workspace on the caller's stream).  The points are the
    ones rhg_sample_points draws for this config (copied to the host beforehand)."""
    n = c["n"]
    a = (c["gamma"] - 1.0) / 2.0
    R = rhg.target_radius(n, c["kbar"], c["gamma"])
    th_d, r_d = rhg.sample_points(n, a, R, seed, device=dev)
    th = torch.empty(n, dtype=torch.float64, pin_memory=True)
    r = torch.empty(n, dtype=torch.float64, pin_memory=True)
    th.copy_(th_d)
    r.copy_(r_d)
    del th_d, r_d
    row_ptr = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    col = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    perm = torch.empty(n, dtype=torch.int32, pin_memory=True)
    bufs = lambda _cap: (row_ptr, col, None, None, None, perm)
    stream = torch.cuda.current_stream()

    def step():
        return rhg._run(lambda o, s: rhg.lib().rhg_generate_from_points(
            n, th.data_ptr(), r.data_ptr(), R, o, s), n, c["fmt"], c["kbar"], device=dev,
            capacity=cap, options=opts, timing=False, workspace=ws, stream=stream,
            host_buffers=True, want_points=False, sample=False, out_bufs=bufs)

    step()
    torch.cuda.synchronize()
    K = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(K):
        g = step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    return {"value": (g.num_edges // 2) / dt, "unit": "edges/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": 16 * n,
            "d2h_bytes_per_step": 8 * (n + 1) + 4 * g.num_edges + (4 * n if args.order == 1 else 0),
            "steps": K, "note": "rhg_generate_from_points, host theta/r in, host CSR out "
                                "(page-locked), wall clock around K calls"}


def measure_e2e(rhg, torch, c, seed, dev, ws, cap, args, opts):
    """Same metric through the public API with HOST (pinned) output buffers: the
    device->host copy of the whole CSR (and of perm for vertex_order 1) is inside
    the timed region.  Inputs are the four scalars (n, kbar, gamma, seed): no
    host->device payload."""
    n = c["n"]
    row_ptr = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    col = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    perm = torch.empty(n, dtype=torch.int32, pin_memory=True)
    bufs = lambda _cap: (row_ptr, col, None, None, None, perm)
    stream = torch.cuda.current_stream()

    def step():
        return rhg._run(lambda o, s: rhg.lib().rhg_generate(n, c["kbar"], c["gamma"], seed, o, s),
                        n, c["fmt"], c["kbar"], device=dev, capacity=cap, options=opts,
                        timing=False, workspace=ws, stream=stream, host_buffers=True,
                        want_points=False, sample=True, out_bufs=bufs)

    step()
    torch.cuda.synchronize()
    K = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(K):
        g = step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / K
    m_und = g.num_edges // 2
    return {"value": m_und / dt, "unit": "edges/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": 8 * (n + 1) + 4 * g.num_edges + (4 * n if args.order == 1 else 0),
            "steps": K, "note": "rhg_generate with host_buffers=1 (page-locked row_ptr/col/perm)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="shard", choices=["replicas", "shard"],
                    help="N > 1: one graph sharded over the ranks (strong scaling, SURVEY "
                         "§8(e); default) or independent graphs per rank (weak)")
    ap.add_argument("--no-configs", action="store_true", help="skip the five-config report")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of graph replay")
    ap.add_argument("--order", type=int, default=0, choices=[0, 1],
                    help="rhg_options.vertex_order of the timed steps (the other is reported too)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dynamic", action="store_true", help="skip the f1 update report")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
