import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_1606_09481_b200 as rhg
for fmt in ("csr",):
    try:
        g = rhg.generate(1_000_000, 32, 2.2, 4, fmt)
        print("ok", g.num_edges)
    except Exception as e:
        print("ERR", e)
