"""d=1 user-order apply with / without the L2 prefetch of v (gp_plan_set_option 3), config 2."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_applies, time_graph
c = W.CONFIGS[2]
x = torch.from_numpy(W.config_points(c)).cuda()
V = torch.randn((100, c.n), dtype=torch.float64, device="cuda"); O = torch.empty_like(V)
s = torch.cuda.current_stream()
for nu2 in (5, 3):
    plan = g.Plan(x, g.Kernel(nu2, c.ell))
    for pf in (0, 1, 0, 1):
        plan.set_option(3, pf)
        mk = lambda st: Applier(g, plan, V, O, st)
        gsec, _ = time_graph(mk, 1000, 5, 1)
        ssec, _ = time_applies(mk(s), 1000, 5, s, 1)
        print(f"nu={nu2}/2 prefetch={pf}: graph {gsec/1000*1e6:.2f} us, stream {ssec/1000*1e6:.2f} us", flush=True)
