"""Generation time per config, eager vs CUDA-graph replay (rhg_options.graph), fixed
output buffers on a non-default stream; device events around each call."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1606_09481_b200 as rhg  # noqa: E402

CFG = {1: (10_000, 6, 3.0, 1, "csr"), 2: (1_000_000, 10, 3.0, 2, "csr"),
       3: (10_000_000, 100, 3.0, 3, "csr"), 4: (1_000_000, 32, 2.2, 4, "csr"),
       5: (100_000_000, 16, 2.7, 5, "pairs")}
s = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with torch.cuda.stream(s):
    for cfg, (n, kbar, gamma, seed, fmt) in CFG.items():
        ws = rhg.Workspace("cuda")
        g = rhg.generate(n, kbar, gamma, seed, fmt, workspace=ws, stream=s)
        cap = g.num_edges
        del g
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda") if fmt == "csr" else None
        col = torch.empty(cap, dtype=torch.int32, device="cuda") if fmt == "csr" else None
        pr = torch.empty((cap, 2), dtype=torch.int32, device="cuda") if fmt != "csr" else None
        out = {"cfg": cfg}
        for mode in (0, 1):
            def run():
                return rhg._run(lambda o, st: rhg.lib().rhg_generate(n, kbar, gamma, seed, o, st),
                                n, fmt, kbar, device="cuda", capacity=cap, options=dict(graph=mode),
                                timing=False, workspace=ws, stream=s, host_buffers=False,
                                want_points=False, sample=True,
                                out_bufs=lambda _c: (rp, col, pr, None, None))
            ms = []
            for i in range(12):
                flush.fill_(i & 0xFF)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                run()
                e1.record(s)
                s.synchronize()
                if i >= 2:
                    ms.append(e0.elapsed_time(e1))
            out["graph" if mode else "eager"] = round(statistics.median(ms), 4)
        print(json.dumps(out))
        del ws, rp, col, pr
        torch.cuda.empty_cache()
