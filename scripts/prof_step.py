"""One rhg_generate step at a BASELINE config, for ncu / timing (not a bench)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1606_09481_b200 as rhg  # noqa: E402

CFG = {1: (10_000, 6, 3.0, 1, "csr"), 2: (1_000_000, 10, 3.0, 2, "csr"),
       3: (10_000_000, 100, 3.0, 3, "csr"), 4: (1_000_000, 32, 2.2, 4, "csr"),
       5: (100_000_000, 16, 2.7, 5, "pairs")}
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fmt", default=None)
ap.add_argument("--heavy", type=int, default=0)
ap.add_argument("--bands", type=int, default=0)
ap.add_argument("--ratio", type=float, default=0.0)
ap.add_argument("--order", type=int, default=0)
ap.add_argument("--graph", type=int, default=0)
a = ap.parse_args()
n, kbar, gamma, seed, fmt = CFG[a.cfg]
fmt = a.fmt or fmt
ws = rhg.Workspace("cuda")
opts = {"heavy_threshold": a.heavy, "num_bands": a.bands, "band_ratio": a.ratio,
        "vertex_order": a.order}
for i in range(a.reps):
    g = rhg.generate(n, kbar, gamma, seed, fmt, workspace=ws, timing=True, options=opts)
    torch.cuda.synchronize()
    t = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in g.timing.items()}
    print(json.dumps({"cfg": a.cfg, "order": a.order, "fmt": fmt, "L": a.bands, "p": a.ratio, "m": g.num_edges, **t}))
