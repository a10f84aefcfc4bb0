"""Profiling driver: config 5 preconditioned CG (rank-400 pivoted Cholesky), a few iterations."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
c5 = W.CONFIGS[5]
x = W.config_points(c5); y = W.config_response(c5, x)
plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(3, c5.ell, form=g.FORM_PRODUCT))
pc = g.Precond(plan, int(sys.argv[1]) if len(sys.argv) > 1 else 400)
yt = torch.from_numpy(y).cuda()
try:
    plan.cg_solve(yt, c5.noise_sigma ** 2, mean=g.MEAN_AFFINE, rtol=1e-8, max_iter=24, precond=pc)
except g.GPError as e:
    print("stopped:", str(e)[:80])
torch.cuda.synchronize()
print("ok")
