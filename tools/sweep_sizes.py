"""Apply time vs N for d = 1, 2, 3 (SURVEY §8(d) scaling sweep: N = 2^14 .. 2^20, x ~ U[0,1]^d,
nu = 3/2, L1, l = 0.1): CUDA-graph timing of back-to-back applies with fresh v."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
from bench import Applier, time_graph

g.use_torch_allocator()
for d in (1, 2, 3):
    for lg in (14, 16, 18, 20):
        n = 1 << lg
        x = torch.from_numpy(W.uniform_points(n, d, 1000 + d)).cuda()
        plan = g.Plan(x, g.Kernel(3, (0.1,) * d))
        nv = max(2, min(32, (1 << 27) // (8 * n)))
        V = torch.randn((nv, n), dtype=torch.float64, device="cuda")
        O = torch.empty_like(V)
        K = 50 if d < 3 else 10
        res = time_graph(lambda s: Applier(g, plan, V, O, s), K, 3, 1, reps=3, stats={})
        us = res[0] / K * 1e6
        print(json.dumps({"d": d, "n": n, "us_per_apply": us, "mvm_per_s": 1e6 / us,
                          "launches": plan.launches_per_apply,
                          "model_gbs": plan.model_bytes / us / 1e3}), flush=True)
        plan.close()
