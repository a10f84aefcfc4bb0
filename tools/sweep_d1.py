"""Time the d=1 apply (CUDA graph of back-to-back applies, fresh v each) for thread-block
shapes given on the command line (default: all), user and rank order, config 2, and check
each shape's output against shape 2 (k_d1_fast 768x9) on the same v."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph

shapes = [int(a) for a in sys.argv[1:]] or list(range(8))
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
nv = 100
V = torch.randn((nv, c.n), dtype=torch.float64, device="cuda")
O = torch.empty_like(V)
for two_nu in (5, 3):
    plan = g.Plan(x, g.Kernel(two_nu, c.ell))
    VR = torch.stack([plan.to_rank(V[i]) for i in range(nv)])
    plan.set_option(1, 2)
    ref_u = plan.kmvm(V[3]).clone()
    ref_r = plan.kmvm_rank(VR[3]).clone()
    for shape in shapes:
        plan.set_option(1, shape)
        eu = (plan.kmvm(V[3]) - ref_u).abs().max().item() / ref_u.abs().max().item()
        er = (plan.kmvm_rank(VR[3]) - ref_r).abs().max().item() / ref_r.abs().max().item()
        row = dict(two_nu=two_nu, shape=shape, relerr_user=eu, relerr_rank=er)
        for rank in (False, True):
            st = {}
            res = time_graph(lambda s: Applier(g, plan, VR if rank else V, O, s, rank_order=rank),
                             100, 5, 1, reps=5, stats=st)
            row["us_rank" if rank else "us_user"] = res[0] / 100 * 1e6
        print(json.dumps(row), flush=True)
    plan.close()
