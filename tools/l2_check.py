"""d=1 config 2 apply time (CUDA graph, 100 applies) vs the number of distinct v / out
buffers cycled: 100 (1.6 GB, inputs from DRAM) down to 2 (L2-resident inputs)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
plan = g.Plan(x, g.Kernel(5, c.ell))
for nv in (100, 16, 4, 2):
    V = torch.randn((nv, c.n), dtype=torch.float64, device="cuda"); O = torch.empty_like(V)
    VR = torch.stack([plan.to_rank(V[i]) for i in range(nv)])
    for rank in (True, False):
        r = time_graph(lambda s: Applier(g, plan, VR if rank else V, O, s, rank_order=rank), 100, 5, 1, reps=5, stats={})
        print(json.dumps(dict(nv=nv, rank=rank, us=r[0] / 100 * 1e6)), flush=True)
