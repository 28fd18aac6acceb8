"""Phase times of rhg_update_moved at config 3 for a few moved fractions (f1)."""
import json
import sys
sys.path.insert(0, '.')
import torch  # noqa: E402
import paper_1606_09481_b200 as rhg  # noqa: E402
n, kbar, gamma, seed = 10_000_000, 100.0, 3.0, 3
a = (gamma - 1) / 2
R = rhg.target_radius(n, kbar, gamma)
th, r = rhg.sample_points(n, a, R, seed)
g0 = rhg.generate_from_points(th, r, R, "csr", kbar_hint=kbar)
tp, tr = rhg.movement_init(n, 103)
FR = [float(x) for x in sys.argv[1:]] or [0.01, 0.05, 0.12]
th1, r1 = th.clone(), r.clone()
rhg.move_points(th1, r1, tp, tr, R, a)
perm = torch.randperm(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
ws = rhg.Workspace("cuda")
for f in FR:
    ids = torch.sort(perm[: int(f * n)]).values
    th_n, r_n = th.clone(), r.clone()
    th_n[ids], r_n[ids] = th1[ids], r1[ids]
    for rep in range(2):
        d = rhg.update_moved(th_n, r_n, R, ids.to(torch.int32), th[ids].contiguous(), r[ids].contiguous(),
                             g0.row_ptr, g0.col, timing=True, workspace=ws)
        t = {k: round(v, 3) if isinstance(v, float) else v for k, v in d.timing.items()}
        print(json.dumps({"frac": f, "rows": d.rows, "removed": len(d.removed), "added": len(d.added), **t}))
