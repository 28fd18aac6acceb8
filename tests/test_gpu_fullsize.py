"""Full-size GPU parity (VERDICT r01 "Prove headline parity on the
full edge set"): the CUDA path, called through the C-ABI exactly as bench.py calls
it (CUDA-graph replay on a dedicated stream), on the ORACLE's points, against the
oracle's complete edge set.

* Config 3 (n = 1e7, kbar = 100, gamma = 3; the headline): every one of the ~1e9
  directed CSR entries and every one of the ~5e8 undirected pairs is compared with
  orc_sweep_csr (rows canonicalised by sorting, SURVEY.md §8(a) output semantics).
* Config 5 (n = 1e8, kbar = 16, gamma = 2.7, pairs): every vertex's degree and
  neighbour-set digest (sum of SplitMix64(w) mod 2^64) against orc_sweep_digest,
  plus 100 complete rows (the 20 innermost vertices, 20 seam straddlers, 60 random)
  against brute force over all 1e8 points.

Disagreements are allowed only on pairs the oracle flags as near ties
(|cosh d - cosh R| <= 1e-12 cosh R, decided in __float128); they are counted and
written to gpurun_out/near_ties.jsonl (committed copies under profiles/)."""
import json
import os
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LOG = os.path.join(ROOT, "gpurun_out", "near_ties.jsonl")
M32 = 0xFFFFFFFF


def record(entry):
    os.makedirs(os.path.dirname(LOG), exist_ok=True)
    with open(LOG, "a") as f:
        f.write(json.dumps(entry) + "\n")
    print(json.dumps(entry))


@pytest.fixture(scope="module")
def rhg():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1606_09481_b200 as rhg
    rhg.lib()
    return rhg


def bench_launch(rhg, th, r, R, fmt):
    """rhg_generate_from_points as bench.py launches rhg_generate: graph mode, a
    dedicated stream, device buffers."""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g = rhg.generate_from_points(th, r, R, fmt, options=dict(graph=1), stream=s)
    s.synchronize()
    return g


def sorted_diff(a, b):
    """Elements of sorted int64 tensor a missing from sorted b (GPU)."""
    if b.numel() == 0:
        return a
    i = torch.searchsorted(b, a).clamp_(max=b.numel() - 1)
    return a[b[i] != a]


def undirected(keys):
    u, v = keys >> 32, keys & M32
    return torch.minimum(u, v) * (1 << 32) + torch.maximum(u, v)


def check_disagreements(only_gpu, only_ref, ties):
    """Every disagreement must be an oracle-flagged near tie; returns the count."""
    tie_keys = {(int(a) << 32) | int(b) for a, b in ties.tolist()}
    dis = torch.cat([undirected(only_gpu), undirected(only_ref)]).unique().cpu().tolist()
    bad = [k for k in dis if k not in tie_keys]
    assert not bad, f"{len(bad)} non-tie disagreements, e.g. {[(k >> 32, k & M32) for k in bad[:5]]}"
    return len(dis)


# --------------------------------------------------------------------------- config 3
@pytest.fixture(scope="module")
def cfg3(orc):
    n, kbar, gamma, seed = 10_000_000, 100.0, 3.0, 3
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    t0 = time.perf_counter()
    csr = orc.sweep_csr(th, r, R, cap_hint=int(1.05 * n * kbar))
    t_orc = time.perf_counter() - t0
    return dict(n=n, R=R, th=th, r=r, csr=csr, t_orc=t_orc)


def oracle_keys_dev(csr, n, dev):
    rp = torch.from_numpy(csr.row_ptr.view(np.int64)).to(dev)
    deg = torch.diff(rp)
    u = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int64), deg)
    col = torch.from_numpy(csr.col.view(np.int32)).to(dev).to(torch.int64) & M32
    return rp, u * (1 << 32) + col


def test_config3_full_csr(rhg, cfg3):
    """All ~1e9 directed entries of config 3 vs orc_sweep_csr (Alg. 1 lines 13-21,
    PAPER.md:157-166; Eq. 3), in the bench's launch configuration."""
    full_csr_compare(rhg, cfg3, {"test": "config3_full_csr"})


def full_csr_compare(rhg, cfg3, tag):
    n, R = cfg3["n"], cfg3["R"]
    dev = torch.device("cuda")
    g = bench_launch(rhg, torch.from_numpy(cfg3["th"]).to(dev), torch.from_numpy(cfg3["r"]).to(dev),
                     R, "csr")
    m = g.num_edges
    gdeg = torch.diff(g.row_ptr)
    gu = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int64), gdeg)
    gk = gu * (1 << 32) + (g.col.to(torch.int64) & M32)
    del gu, gdeg
    assert not bool(((gk >> 32) == (gk & M32)).any()), "self-loop"
    gk = torch.sort(gk).values
    del g
    torch.cuda.empty_cache()
    assert bool((gk[1:] != gk[:-1]).all()), "duplicate entries"
    # symmetry: the transposed key set is the same set
    tk = torch.sort((gk & M32) * (1 << 32) + (gk >> 32)).values
    assert torch.equal(tk, gk), "CSR not symmetric"
    del tk
    orp, ok = oracle_keys_dev(cfg3["csr"], n, dev)
    same = m == ok.numel() and torch.equal(gk, ok)
    excused = 0
    if not same:
        excused = check_disagreements(sorted_diff(gk, ok), sorted_diff(ok, gk), cfg3["csr"].ties)
    record({**tag, "n": n, "directed_entries": int(m),
            "oracle_directed_entries": int(ok.numel()), "oracle_near_tie_pairs": len(cfg3["csr"].ties),
            "disagreements": excused, "excused_as_near_ties": excused,
            "oracle_seconds": round(cfg3["t_orc"], 1)})


def test_config3_full_pairs(rhg, cfg3):
    """All ~5e8 undirected (u < v) pairs of config 3 vs the oracle's edge set."""
    n, R = cfg3["n"], cfg3["R"]
    dev = torch.device("cuda")
    g = bench_launch(rhg, torch.from_numpy(cfg3["th"]).to(dev), torch.from_numpy(cfg3["r"]).to(dev),
                     R, "pairs")
    P = g.pairs.to(torch.int64) & M32
    assert bool((P[:, 0] < P[:, 1]).all())
    gk = torch.sort(P[:, 0] * (1 << 32) + P[:, 1]).values
    del P, g
    torch.cuda.empty_cache()
    assert bool((gk[1:] != gk[:-1]).all()), "duplicate undirected edge"
    _, ok = oracle_keys_dev(cfg3["csr"], n, dev)
    ok = ok[(ok >> 32) < (ok & M32)]  # rows ascending, columns ascending: already sorted
    same = torch.equal(gk, ok)
    excused = 0
    if not same:
        excused = check_disagreements(sorted_diff(gk, ok), sorted_diff(ok, gk), cfg3["csr"].ties)
    record({"test": "config3_full_pairs", "n": n, "undirected_edges": int(gk.numel()),
            "oracle_undirected_edges": int(ok.numel()),
            "oracle_near_tie_pairs": len(cfg3["csr"].ties), "disagreements": excused,
            "excused_as_near_ties": excused})


EXTRA = [tuple(float(x) for x in c.split(",")) for c in
         os.environ.get("RHG_FULLSIZE_EXTRA", "").split(";") if c.strip()]


def _full_csr_other_seeds(rhg, orc, case):
    """The config-3 comparison (all directed entries, bench launch configuration) on
    other seeds / parameters at full scale; opt-in because each case costs the oracle
    about half a minute.  Logged results: profiles/r02_near_ties.jsonl."""
    n, kbar, gamma, seed = int(case[0]), case[1], case[2], int(case[3])
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    t0 = time.perf_counter()
    csr = orc.sweep_csr(th, r, R, cap_hint=int(1.05 * n * kbar))
    full_csr_compare(rhg, dict(n=n, R=R, th=th, r=r, csr=csr, t_orc=time.perf_counter() - t0),
                     {"test": "full_csr_other_seeds", "kbar": kbar, "gamma": gamma, "seed": seed})


if EXTRA:  # opt-in (RHG_FULLSIZE_EXTRA='n,kbar,gamma,seed;...'): not collected otherwise
    test_full_csr_other_seeds = pytest.mark.parametrize("case", EXTRA)(_full_csr_other_seeds)


# --------------------------------------------------------------------------- config 5
def mix64_dev(w):
    """SplitMix64 finaliser on int64 tensors (wrapping arithmetic; logical shifts)."""
    def srl(z, k):
        return (z >> k) & ((1 << (64 - k)) - 1)
    c = lambda x: x - (1 << 64) if x >= (1 << 63) else x
    z = w * c(0x9E3779B97F4A7C15) + c(0x632BE59BD9B4E019)
    z = (z ^ srl(z, 30)) * c(0xBF58476D1CE4E5B9)
    z = (z ^ srl(z, 27)) * c(0x94D049BB133111EB)
    return z ^ srl(z, 31)


def test_config5_full_digest_and_rows(rhg, orc):
    """Config 5 (n = 1e8, pairs) on the oracle's points: every vertex's degree and
    neighbour digest vs orc_sweep_digest; then 100 complete rows vs brute force."""
    n, kbar, gamma, seed = 100_000_000, 16.0, 2.7, 5
    a = orc.alpha(gamma)
    R = orc.target_radius(n, kbar, a)
    th, r = orc.sample_points(n, a, R, seed)
    dev = torch.device("cuda")
    g = bench_launch(rhg, torch.from_numpy(th).to(dev), torch.from_numpy(r).to(dev), R, "pairs")
    P = g.pairs
    m = g.num_edges
    assert bool((P[:, 0].to(torch.int64) & M32 < P[:, 1].to(torch.int64) & M32).all())
    deg = torch.zeros(n, dtype=torch.int64, device=dev)
    dig = torch.zeros(n, dtype=torch.int64, device=dev)
    step = 1 << 26
    for s0 in range(0, m, step):
        u = P[s0:s0 + step, 0].to(torch.int64) & M32
        v = P[s0:s0 + step, 1].to(torch.int64) & M32
        one = torch.ones_like(u)
        deg.index_add_(0, u, one)
        deg.index_add_(0, v, one)
        dig.index_add_(0, u, mix64_dev(v))
        dig.index_add_(0, v, mix64_dev(u))
        del u, v, one
    t0 = time.perf_counter()
    om, odeg, odig, ties, _ = orc.sweep_digest(th, r, R)
    t_orc = time.perf_counter() - t0
    gdeg = deg.cpu().numpy().astype(np.uint64)
    gdig = dig.cpu().numpy().view(np.uint64)
    bad_v = np.nonzero((gdeg != odeg) | (gdig != odig))[0]
    tie_v = set(ties.ravel().tolist())
    assert set(bad_v.tolist()) <= tie_v, f"vertices {bad_v[:10]} differ outside the near-tie set"

    def row(v):
        vv = torch.tensor(int(v), dtype=torch.int64, device=dev)
        pu = P[:, 0].to(torch.int64) & M32
        pv = P[:, 1].to(torch.int64) & M32
        return torch.cat([pv[pu == vv], pu[pv == vv]]).cpu().numpy().astype(np.uint32)

    rng = np.random.default_rng(5)
    order = np.argsort(th)
    q = np.unique(np.concatenate([np.argsort(r)[:20], order[:10], order[-10:],
                                  rng.choice(n, 60, replace=False)])).astype(np.uint32)
    q = np.unique(np.concatenate([q, bad_v.astype(np.uint32)]))
    off, nbr, _ = orc.rows(th, r, R, q)
    excused = 0
    for k, v in enumerate(q):
        ref = nbr[off[k]:off[k + 1]]
        got = np.sort(row(v))
        if not np.array_equal(got, ref):
            diff = np.setxor1d(got, ref)
            w, _ = orc.row_ties(th, r, R, int(v))
            assert set(diff.tolist()) <= set(w.tolist()), f"vertex {v}: {diff[:10]}"
            excused += len(diff)
    assert m == om or len(bad_v) > 0
    record({"test": "config5_full_digest_and_rows", "n": n, "undirected_edges": int(m),
            "oracle_undirected_edges": int(om), "oracle_near_tie_pairs": int(len(ties)),
            "vertices_with_digest_mismatch": int(len(bad_v)), "exact_rows_checked": int(len(q)),
            "row_disagreements_excused_as_near_ties": excused,
            "oracle_digest_seconds": round(t_orc, 1)})
