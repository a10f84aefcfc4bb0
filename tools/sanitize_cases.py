"""Small cases through every kernel path (for compute-sanitizer runs)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2508_01864_b200 as g
rng = np.random.default_rng(0)
for d, n, form, two_nu in [(1, 3000, 0, 5), (2, 3000, 0, 3), (2, 2500, 1, 3), (3, 2100, 0, 5)]:
    x = torch.from_numpy(rng.random((n, d))).cuda()
    plan = g.Plan(x, g.Kernel(two_nu, (0.1, 0.2, 0.3)[:d], form=form))
    V = torch.randn((3, n), dtype=torch.float64, device="cuda")
    plan.kmvm(V)
    plan.kmvm_rank(plan.to_rank(V[0]))
    z = torch.from_numpy(rng.random((300, d))).cuda()
    plan.cross(z).kzx(V[0].contiguous())
    if d == 1:
        plan.set_option(0, 2); plan.kmvm(V[1].contiguous()); plan.set_option(0, 0)
        plan.set_option(0, 3); plan.kmvm(V); plan.kmvm_rank(plan.to_rank(V[0]))   # path 3
        plan.kmvm_dlengthscale(V[1].contiguous()); plan.set_option(0, 0)
        plan.kmvm_dlengthscale(V)
    if form == 1 or d == 1:
        y = torch.randn(n, dtype=torch.float64, device="cuda")
        plan.cg_solve(y, 0.1, mean=g.MEAN_AFFINE, rtol=1e-6, max_iter=200)
torch.cuda.synchronize()
print("sanitize cases ok")
