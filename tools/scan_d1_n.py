import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle
import paper_2508_01864_b200 as g
rng = np.random.default_rng(3)
ns = [1296, 1727, 1940, 2294, 2582, 4404, 4690, 4845] + list(range(1025, 5300, 61))
bad = []
for n in ns:
    x = rng.random((n, 1)); v = rng.standard_normal(n)
    plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(3, (0.1,), 1.0))
    out = plan.kmvm(torch.from_numpy(v).cuda()).cpu().numpy()
    ref, ab = oracle.kmvm_rows(x, v, 3, "l1", (0.1,), 1.0, return_abs=True)
    err = np.abs(out - ref) / (ab.max() * np.abs(v).max())
    outr = plan.from_rank(plan.kmvm_rank(plan.to_rank(torch.from_numpy(v).cuda()))).cpu().numpy()
    errr = np.abs(outr - ref) / (ab.max() * np.abs(v).max())
    if err.max() > 1e-9 or errr.max() > 1e-9:
        order = np.argsort(x[:, 0], kind="stable"); rank = np.empty(n, int); rank[order] = np.arange(n)
        br = np.sort(rank[np.nonzero(err > 1e-9)[0]])
        bad.append(n)
        print(f"n={n} user err {err.max():.2e} ({len(br)} rows, ranks {br[:6]}..{br[-3:]}) rank-order err {errr.max():.2e}", flush=True)
    plan.close()
print("bad n:", bad)
