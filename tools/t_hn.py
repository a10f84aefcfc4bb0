import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2508_01864_b200 as g
case = sys.argv[1]
d, nu, n = [int(v) for v in case.split(",")]
x = np.random.default_rng(0).random((n, d))
plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu, (0.1,) * d))
try:
    out = plan.kmvm(torch.ones(n, dtype=torch.float64, device="cuda"))
    torch.cuda.synchronize()
    print(case, "ok", out[:2].tolist())
except Exception as e:
    print(case, "FAIL", str(e)[:200])
