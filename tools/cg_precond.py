"""Config-5 CG (4 RHS, product-3/2, N=3e5, rtol 1e-8): unpreconditioned vs pivoted-Cholesky
preconditioned (gp_cg_solve_pc) for several ranks; setup / solve times and iterations."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
c = W.CONFIGS[5]
x = W.config_points(c); y = W.config_response(c, x)
plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(3, c.ell, form=g.FORM_PRODUCT))
yt = torch.from_numpy(y).cuda()
ranks = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 100, 200, 400]
for rank in ranks:
    pc = None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if rank:
        pc = g.Precond(plan, rank)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    a, b, info = plan.cg_solve(yt, c.noise_sigma ** 2, mean=g.MEAN_AFFINE, rtol=1e-8,
                               max_iter=40000, precond=pc)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"rank {rank}: precond setup {t1 - t0:.3f} s, solve {t2 - t1:.3f} s, iters {info['iters']}, "
          f"relres {info['relres_max']:.2e}, restarts {info['restarts']}, beta {[round(v, 5) for v in b]}",
          flush=True)
    if pc:
        pc.close()
