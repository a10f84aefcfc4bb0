import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2508_01864_b200 as g
import oracle
for n in [int(a) for a in sys.argv[1:]]:
    x = np.random.default_rng(1).random((n, 3))
    v = np.random.default_rng(2).standard_normal(n)
    plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(5, (0.2, 0.3, 0.5)))
    out = plan.kmvm(torch.from_numpy(v).cuda()).cpu().numpy()
    rows = np.random.default_rng(3).choice(n, 200, replace=False)
    ref, ab = oracle.kmvm_rows(x, v, 5, "l1", (0.2, 0.3, 0.5), rows=rows, return_abs=True)
    err = np.abs(out[rows] - ref).max()
    print(n, plan.levels, f"err={err:.3e} tol={1e-9*ab.max()*np.abs(v).max():.3e}", "BAD" if err > 1e-9*ab.max()*np.abs(v).max() else "ok", flush=True)
