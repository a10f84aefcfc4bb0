"""d = 1 apply time vs N (CUDA graph of back-to-back applies, fresh v), user and rank order:
single-chunk k_d1_ov up to #SMs x 6912 points, multi-sub-tile k_d1_coop above."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph

for n in [1 << 16, 1 << 18, 1_000_000, 1 << 20, 1 << 21, 1 << 22, 1 << 23]:
    x = torch.from_numpy(W.uniform_points(n, 1, 7)).cuda()
    nv = max(2, min(64, (1 << 27) // (8 * n)))
    V = torch.randn((nv, n), dtype=torch.float64, device="cuda")
    O = torch.empty_like(V)
    plan = g.Plan(x, g.Kernel(5, (0.05,)))
    VR = torch.stack([plan.to_rank(V[i]) for i in range(nv)])
    row = {"n": n, "path": plan.query(6)}
    for rank in (False, True):
        K = 50
        res = time_graph(lambda s: Applier(g, plan, VR if rank else V, O, s, rank_order=rank), K, 3, 1, reps=3, stats={})
        us = res[0] / K * 1e6
        row["us_rank" if rank else "us_user"] = us
        row["gbs_rank" if rank else "gbs_user"] = (24 if rank else 28) * n / us / 1e3
    print(json.dumps(row), flush=True)
    plan.close()
