"""Apply timing of the d >= 2 path on configs 3-5 (engine A/B history: profiles/r01_notes.md)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2508_01864_b200 as g
import workloads as W


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


cases = [(3, 3, 0, 1, False), (5, 3, 1, 4, True), (5, 3, 1, 1, True), (4, 5, 0, 1, False)]
if len(sys.argv) > 1:
    cases = [cases[int(i)] for i in sys.argv[1].split(",")]
for cfg, nu2, form, nrhs, rank in cases:
    c = W.CONFIGS[cfg]
    x = torch.from_numpy(W.config_points(c)).cuda()
    plan = g.Plan(x, g.Kernel(nu2, c.ell, form=form))
    V = torch.from_numpy(np.stack([W.config_vector(c, j) for j in range(nrhs)])).cuda()
    if nrhs == 1:
        V = V[0]
    O = torch.empty_like(V)
    f = (lambda: plan.kmvm_rank(V, O)) if rank else (lambda: plan.kmvm(V, O))
    ms = timeit(f, 10 if cfg != 4 else 3)
    print(f"config {cfg} nu={nu2}/2 form={form} nrhs={nrhs} rank={rank}: "
          f"{ms * 1e3:.1f} us / apply", flush=True)
