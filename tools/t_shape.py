"""d = 1 apply time around the single-chunk capacity for each thread-block shape
(GPM_D1_SHAPE: 0 = 256 x 3x9, 1 = 256 x 3x10, 2 = 256 x 4x7)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph

for n in [1_000_000, 1_022_976, 1_030_000, 1 << 20, 1_060_864]:
    x = torch.from_numpy(W.uniform_points(n, 1, 7)).cuda()
    V = torch.randn((16, n), dtype=torch.float64, device="cuda")
    O = torch.empty_like(V)
    for shape in (-1, 0, 1, 2):
        plan = g.Plan(x, g.Kernel(3, (0.1,)))
        if shape >= 0:
            try:
                plan.set_option(1, shape)
            except Exception as e:
                print(n, shape, "set_option failed", e); continue
        row = {"n": n, "shape": shape, "path": plan.query(6)}
        for rank in (False, True):
            res = time_graph(lambda s: Applier(g, plan, V, O, s, rank_order=rank), 50, 3, 1, reps=3, stats={})
            row["us_rank" if rank else "us_user"] = round(res[0] / 50 * 1e6, 2)
        print(json.dumps(row), flush=True)
        plan.close()
