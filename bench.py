#!/usr/bin/env python
"""Benchmark: threshold RHG generation (arXiv 1606.09481, Algorithm 1) on B200.

Default workload = BASELINE.json configs[2] ("config 3", the headline metric):
n = 1e7, kbar = 100, gamma = 3 (alpha = 1), Philox seed 3, CSR (uint64 row_ptr,
uint32 col).  One step = one rhg_generate call: sampling, band assignment, sort,
index, range queries with exact tests, count -> scan -> emit (every step of the
hot path, nothing cached).  Output buffers and workspace are preallocated.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  N > 1 (torchrun): every rank generates its own
independent graph (seed 3 + rank): replicas, weak scaling, no data-path collective.
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
FP64_OPS_PER_TEST = 14  # certified predicate: 11 DMUL/DADD + 2 DFMA... see DESIGN.md


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


def oracle_sample_run(frac: float):
    """One bounded sample of the config-3 workload on the CPU oracle: sample all n
    points (Philox + inverse CDF), sort by angle, sweep the vertices with id in
    [0, frac*n).  Returns (undirected edges found, seconds, tests)."""
    import oracle
    c = CONFIG3
    t0 = time.perf_counter()
    a = oracle.alpha(c["gamma"])
    R = oracle.target_radius(c["n"], c["kbar"], a)
    th, r = oracle.sample_points(c["n"], a, R, c["seed"])
    m, tests = oracle.sweep_count(th, r, R, 0, int(frac * c["n"]))
    return m, time.perf_counter() - t0, tests


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    frac = args.ref_frac
    for _ in range(args.warmup if args.warmup < 1 else 1):
        oracle_sample_run(frac / 4)
    vals, secs, ms = [], [], []
    for _ in range(args.steps):
        m, s, _t = oracle_sample_run(frac)
        vals.append(m / s)
        secs.append(s)
        ms.append(m)
    value = sum(ms) / sum(secs)
    sample = (f"per step: all {CONFIG3['n']} points sampled + angle-sorted, edges found from the "
              f"vertices with id < {int(frac * CONFIG3['n'])} ({frac:.3f} of the queries); "
              f"value = edges found / wall time")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Philox-sampled points, seed 3)",
            "config": {"workload": WORKLOAD, "n": CONFIG3["n"], "kbar": CONFIG3["kbar"],
                       "gamma": CONFIG3["gamma"], "format": "count only"},
            "cpu_baseline": {"value": value, "unit": "edges/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
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
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    c = CONFIG3
    seed = c["seed"] + rank
    stream = torch.cuda.current_stream()
    ws = rhg.Workspace(dev)

    # warm-up: also sizes the output exactly (capacity protocol)
    g = rhg.generate(c["n"], c["kbar"], c["gamma"], seed, c["fmt"], device=dev, workspace=ws)
    cap = g.num_edges
    row_ptr = torch.empty(c["n"] + 1, dtype=torch.int64, device=dev)
    col = torch.empty(cap, dtype=torch.int32, device=dev)
    del g
    bufs = lambda _cap: (row_ptr, col, None, None, None)

    def step(timing=False):
        return rhg._run(lambda o, s: rhg.lib().rhg_generate(c["n"], c["kbar"], c["gamma"], seed, o, s),
                        c["n"], c["fmt"], c["kbar"], device=dev, capacity=cap, options=None,
                        timing=timing, workspace=ws, stream=stream, host_buffers=False,
                        want_points=False, sample=True, out_bufs=bufs)

    for _ in range(args.warmup):
        step()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phases = []
    clk = ClockSampler(local)
    clk.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    last = None
    for i in range(args.steps):
        flush.fill_(i & 0xFF)  # L2 flush between timed steps, outside the events
        ev[i][0].record(stream)
        last = step(timing=True)
        ev[i][1].record(stream)
        phases.append(last.timing)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clocks = clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    edges = torch.tensor([float(last.num_edges // 2)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(edges, op=dist.ReduceOp.SUM)
    tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    m_und_total = float(edges.item())  # undirected edges per step, all ranks
    value = m_und_total / (ms_per_step * 1e-3)

    # per-phase device times (events on this stream, inside the timed steps)
    keys = ["ms_sample", "ms_sort", "ms_index", "ms_count", "ms_scan", "ms_emit"]
    ph = {k: statistics.median([p[k] for p in phases]) for k in keys}
    cand = phases[-1]["candidates"]
    launches = int(sum(p["launches"] for p in phases))
    n = c["n"]
    m_dir = last.num_edges
    P = peaks()
    hbm_peak = P.get("hbm_gbs", 6650.0)
    # emit pass: algorithmic bytes = col (4 B / directed edge) + row_ptr read (8 B / vertex)
    #            + query SoA read once (32 B / point) + sid gather (4 B / directed edge)
    emit_bytes = 4 * m_dir + 8 * (n + 1) + 32 * n + 4 * m_dir
    count_ops = FP64_OPS_PER_TEST * cand
    count_s, emit_s = ph["ms_count"] * 1e-3, ph["ms_emit"] * 1e-3
    roof_count = {"kernel": "k_query<COUNT>", "bound": "alu", "achieved": count_ops / count_s / 1e12,
                  "peak": FP64_PEAK_OPS / 1e12, "unit": "TFLOP/s (fp64 ops)",
                  "frac": count_ops / count_s / FP64_PEAK_OPS, "traffic": None,
                  "peak_source": "measured DFMA rate, profiles/r01_fp64_microbench.txt"}
    roof_emit = {"kernel": "k_query<EMIT>", "bound": "hbm", "achieved": emit_bytes / emit_s / 1e9,
                 "peak": hbm_peak, "unit": "GB/s", "frac": emit_bytes / emit_s / 1e9 / hbm_peak,
                 "traffic": None, "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}
    dominant = roof_count if count_s >= emit_s else roof_emit
    # north-star convention: points read (32 B) + 8 B per emitted directed edge, over query+emit
    ns_bytes = 32 * n + 8 * m_dir
    qe_s = count_s + ph["ms_scan"] * 1e-3 + emit_s
    north_star = {"query_emit_ms": qe_s * 1e3, "bytes": ns_bytes,
                  "GBps": ns_bytes / qe_s / 1e9, "frac_of_measured": ns_bytes / qe_s / 1e9 / hbm_peak,
                  "frac_of_8TBps": ns_bytes / qe_s / 1e9 / 8000.0}

    e2e = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_e2e:
        e2e = measure_e2e(rhg, torch, c, seed, dev, ws, cap, args)
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        m_s, s_s, tests = oracle_sample_run(args.cpu_frac)
        cpu = {"value": m_s / s_s, "unit": "edges/s", "cores": oracle.num_threads(),
               "kind": "oracle",
               "sample": (f"all {n} points sampled + angle-sorted, sweep over vertices with "
                          f"id < {int(args.cpu_frac * n)} ({args.cpu_frac:.3f} of queries): "
                          f"{m_s} edges, {tests} tests in {s_s:.2f} s"),
               "cpu": cpu_model()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (Philox4x32-10-sampled points, seed 3 + rank)",
                "config": {"workload": WORKLOAD, "n": n, "kbar": c["kbar"], "gamma": c["gamma"],
                           "format": "csr", "parallelism": "replicas" if world > 1 else "single",
                           "l2": "flushed between steps (256 MiB fill outside the step events)",
                           "undirected_edges_per_step_per_rank": m_dir // 2},
                "roofline": dominant, "roofline_other": roof_emit if dominant is roof_count else roof_count,
                "north_star_hbm": north_star,
                "phases_ms": ph, "candidates": cand,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "wall_s_timed_loop": wall,
                "library": rhg.version()}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(rhg, torch, c, seed, dev, ws, cap, args):
    """Same metric through the public API with HOST (pinned) output buffers: the
    device->host copy of the whole CSR is inside the timed region.  Inputs are the
    four scalars (n, kbar, gamma, seed): no host->device payload."""
    n = c["n"]
    row_ptr = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
    col = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    bufs = lambda _cap: (row_ptr, col, None, None, None)
    stream = torch.cuda.current_stream()

    def step():
        return rhg._run(lambda o, s: rhg.lib().rhg_generate(n, c["kbar"], c["gamma"], seed, o, s),
                        n, c["fmt"], c["kbar"], device=dev, capacity=cap, options=None,
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
            "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8 * (n + 1) + 4 * g.num_edges,
            "steps": K, "note": "rhg_generate with host_buffers=1 (page-locked row_ptr/col)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-frac", type=float, default=0.05)
    ap.add_argument("--ref-frac", type=float, default=0.02)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
