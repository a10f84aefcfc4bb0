"""Timing driver: config-5 pivoted-Cholesky preconditioner setup (gp_precond_create) at
several ranks, twice each (the first includes cuBLAS handle creation / lazy loading)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
c5 = W.CONFIGS[5]
x = W.config_points(c5)
plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(3, c5.ell, form=g.FORM_PRODUCT))
for rank in [1, 1, 100, 400, 400]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pc = g.Precond(plan, rank)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pc.close()
    print(f"rank {rank}: {1e3 * (t1 - t0):.1f} ms")
