"""Quick parity + timing of the d >= 2 bench algebras (experiment builds: GPM_LIB=...)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2508_01864_b200 as g


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
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


rng = np.random.default_rng(5)
bad = 0
for d, nu2, form, ell, n, nrhs in [(2, 3, 0, (0.1, 0.2), 5000, 1), (2, 3, 0, (0.1, 0.2), 70001, 1),
                                   (2, 3, 1, (0.1, 0.1), 70001, 4), (3, 5, 0, (0.2, 0.3, 0.5), 3000, 1),
                                   (3, 5, 0, (0.2, 0.3, 0.5), 70001, 1), (3, 5, 0, (0.2, 0.3, 0.5), 1 << 14, 1)]:
    x = rng.random((n, d)); V = rng.standard_normal((nrhs, n))
    plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu2, ell, 1.0, form))
    Vd = torch.from_numpy(V).cuda()
    out = plan.kmvm(Vd if nrhs > 1 else Vd[0]).cpu().numpy().reshape(nrhs, n)
    rows = rng.choice(n, 256, replace=False)
    worst = 0.0
    for c in range(nrhs):
        ref, ab = oracle.kmvm_rows(x, V[c], nu2, ["l1", "product"][form], ell, 1.0, rows=rows,
                                   return_abs=True)
        worst = max(worst, np.max(np.abs(out[c][rows] - ref)) / (ab.max() * np.abs(V[c]).max()))
    vv = Vd if nrhs > 1 else Vd[0]
    o = torch.empty_like(vv)
    us = timeit(lambda: plan.kmvm(vv, o)) * 1e3
    ok = worst <= 1e-9
    bad += not ok
    print(f"d={d} nu={nu2}/2 form={form} n={n} nrhs={nrhs}: rel err {worst:.2e} {'ok' if ok else 'FAIL'}  {us:.1f} us", flush=True)
    plan.close()
print("exp_check", "FAILED" if bad else "passed")
