"""Timing driver: d = 2 product-form applies at config-3 size (N = 2e5, l = (0.1, 0.2)) for
nu = 3/2 .. 9/2, K v and (nu <= 7/2) the lengthscale-gradient MVM; CUDA events, 20 applies."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2508_01864_b200 as g
rng = np.random.default_rng(0)
n = 200000
x = torch.from_numpy(rng.random((n, 2))).cuda()
v = torch.from_numpy(rng.standard_normal(n)).cuda()
for two_nu in [3, 5, 7, 9]:
    plan = g.Plan(x, g.Kernel(two_nu, (0.1, 0.2), 1.0, form=g.FORM_PRODUCT))
    res = {}
    for name, fn in [("kmvm", plan.kmvm), ("dlengthscale", plan.kmvm_dlengthscale)]:
        if name == "dlengthscale" and two_nu == 9:
            continue
        fn(v); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn(v)
        e1.record(); torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 20 * 1e3, 1)
    print(f"product nu={two_nu}/2 N={n}: us per apply {res}", flush=True)
    plan.close()
