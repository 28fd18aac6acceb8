import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_1606_09481_b200 as rhg
opts = dict(num_bands=int(sys.argv[1]), band_ratio=float(sys.argv[2])) if len(sys.argv) > 2 else None
fmt = sys.argv[3] if len(sys.argv) > 3 else "csr"
n, kbar, gamma, seed = 20_000, 12, 2.4, 17
a = oracle.alpha(gamma); R = oracle.target_radius(n, kbar, a); th, r = oracle.sample_points(n, a, R, seed)
g = rhg.generate_from_points(torch.from_numpy(th).cuda(), torch.from_numpy(r).cuda(), R, fmt, options=opts, timing=True)
torch.cuda.synchronize()
print("ok", opts, fmt, g.num_edges, g.timing)
