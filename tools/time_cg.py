"""Config-5 CG timing (4 RHS, product Matern-3/2, N = 3e5, rtol 1e-8): fused / graph
(default), fused without graph (GPM_CG_NOGRAPH), unfused (GPM_CG_UNFUSED) -- run each in
its own process: python tools/time_cg.py"""
import os, sys, json, time, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) == 1:
    for env in ({}, {"GPM_CG_NOGRAPH": "1"}, {"GPM_CG_UNFUSED": "1"}):
        subprocess.run([sys.executable, __file__, "run"], env={**os.environ, **env})
    sys.exit(0)
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
c = W.CONFIGS[5]
x = W.config_points(c); y = W.config_response(c, x)
g.use_torch_allocator()
plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(3, c.ell, form=g.FORM_PRODUCT))
yd = torch.from_numpy(y).cuda()
try:
    plan.cg_solve(yd, c.noise_sigma ** 2, rtol=1e-8, max_iter=64)   # warm-up
except g.GPError:
    pass
torch.cuda.synchronize()
t = time.perf_counter()
a, b, info = plan.cg_solve(yd, c.noise_sigma ** 2, rtol=1e-8, max_iter=40000)
torch.cuda.synchronize()
t = time.perf_counter() - t
mode = "unfused" if os.environ.get("GPM_CG_UNFUSED") else ("fused, no graph" if os.environ.get("GPM_CG_NOGRAPH") else "fused + graph")
print(json.dumps(dict(mode=mode, s=t, iters=info["iters"], ms_per_iter=t / info["iters"] * 1e3,
                      relres=info["relres_max"], beta=b)), flush=True)
