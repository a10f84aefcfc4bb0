"""Graph / stream per-apply time of the d=1 kernel with and without PDL (config 2)."""
import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_applies, time_graph
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
V = torch.randn((64, c.n), dtype=torch.float64, device="cuda"); O = torch.empty_like(V)
s = torch.cuda.current_stream()
for nu2 in (5, 3):
    plan = g.Plan(x, g.Kernel(nu2, c.ell))
    VR = torch.stack([plan.to_rank(V[i]) for i in range(64)])
    for pdl in (0, 1):
        plan.set_option(2, pdl)
        for rank in (False, True):
            mk = lambda st: Applier(g, plan, VR if rank else V, O, st, rank_order=rank)
            gsec, _ = time_graph(mk, 1000, 5, 1)
            ssec, _ = time_applies(mk(s), 1000, 5, s, 1)
            print(f"nu={nu2}/2 pdl={pdl} rank={rank}: graph {gsec/1000*1e6:.2f} us, stream {ssec/1000*1e6:.2f} us", flush=True)
