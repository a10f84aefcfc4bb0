"""Apply time of the d = 3 product form ((p+1)^2 sub-passes per level) next to the L1 form."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2508_01864_b200 as g
import workloads as W

c = W.CONFIGS[4]
x = torch.from_numpy(W.config_points(c)).cuda()
v = torch.from_numpy(W.config_vector(c, 0)).cuda()
for nu2 in (1, 3, 5, 7, 9):
    for form in (0, 1):
        plan = g.Plan(x, g.Kernel(nu2, c.ell, form=form))
        o = torch.empty_like(v)
        plan.kmvm(v, o); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            plan.kmvm(v, o)
        e1.record(); torch.cuda.synchronize()
        print(f"config-4 points (n=5e5, d=3) nu={nu2}/2 form={'product' if form else 'L1'}: "
              f"{e0.elapsed_time(e1) / reps:.2f} ms / apply", flush=True)
        plan.close()
