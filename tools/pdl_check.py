import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
V = torch.randn((100, c.n), dtype=torch.float64, device="cuda"); O = torch.empty_like(V)
plan = g.Plan(x, g.Kernel(5, c.ell))
VR = torch.stack([plan.to_rank(V[i]) for i in range(100)])
for pdl in (1, 0):
    plan.set_option(2, pdl)
    for rank in (True, False):
        r = time_graph(lambda s: Applier(g, plan, VR if rank else V, O, s, rank_order=rank), 100, 5, 1, reps=5, stats={})
        print(json.dumps(dict(pdl=pdl, rank=rank, us=r[0] / 100 * 1e6)), flush=True)
