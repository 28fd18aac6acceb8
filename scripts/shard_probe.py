"""Per-shard visited candidates (tests + certain) of one config: shard balance."""
import sys
sys.path.insert(0, '.')
import paper_1606_09481_b200 as rhg  # noqa: E402
CFG = {2: (1_000_000, 10, 3.0, 2), 4: (1_000_000, 32, 2.2, 4)}
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32
fmt = sys.argv[3] if len(sys.argv) > 3 else "csr"
n, kbar, gamma, seed = CFG[cfg]
rows = []
for s in range(N):
    g = rhg.generate(n, kbar, gamma, seed, fmt, timing=True, options=dict(shard_index=s, shard_count=N))
    t = g.timing
    act = t["candidates"] + t["certain"]
    rows.append((s, act, t["candidates"], t["certain"], g.num_edges))
mean = sum(r[1] for r in rows) / N
for r in rows:
    print(fmt, cfg, N, "shard %d candidates %d (%.3f of mean) tests %d certain %d edges %d"
          % (r[0], r[1], r[1] / mean, r[2], r[3], r[4]))
