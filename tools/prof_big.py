"""Profiling driver: d = 1 reduce-then-scan path at N = 2^23 (a few applies)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2508_01864_b200 as g
import workloads as W
n = 1 << 23
x = torch.from_numpy(W.uniform_points(n, 1, 7)).cuda()
plan = g.Plan(x, g.Kernel(5, (0.05,)))
v = torch.randn(n, dtype=torch.float64, device="cuda")
vr = plan.to_rank(v)
for _ in range(3):
    plan.kmvm(v)
    plan.kmvm_rank(vr)
torch.cuda.synchronize()
print("ok", plan.d1_path)
