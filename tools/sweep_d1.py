"""Time the d=1 apply for every thread-block shape, user and rank order (config 2)."""
import os, sys, ctypes, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
sys.path.insert(0, ROOT)
from bench import Applier, time_applies, per_launch

c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
nv = 64
V = torch.randn((nv, c.n), dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
s = torch.cuda.current_stream()
res = []
for two_nu in (3, 5):
    plan = g.Plan(x, g.Kernel(two_nu, c.ell))
    VR = torch.stack([plan.to_rank(V[i]) for i in range(nv)])
    for shape in range(4):
        plan.set_option(1, shape)
        for rank in (False, True):
            ap = Applier(g, plan, VR if rank else V, O, s, rank_order=rank)
            sec, _ = time_applies(ap, 1000, 10, s, 1)
            m, med, mn = per_launch(ap, 200, s)
            res.append(dict(two_nu=two_nu, shape=shape, rank=rank, us_loop=sec / 1000 * 1e6,
                            us_launch_med=med * 1e6, us_min=mn * 1e6))
            print(json.dumps(res[-1]), flush=True)
