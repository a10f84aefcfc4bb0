"""gp_kmvm_host (host buffers, pipelined copies) equals gp_kmvm on device buffers, bitwise, for
random plans and column counts; repeated calls on one plan (slot reuse).  One-off check."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2508_01864_b200 as g
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
for it in range(60):
    d = int(rng.integers(1, 4)); nu2 = int(rng.choice([1, 3, 5])); form = int(rng.integers(0, 2))
    n = int(rng.integers(1, 200000 if d == 1 else 20000))
    x = rng.random((n, d))
    plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu2, tuple(10 ** rng.uniform(-1.5, 0, d)), 1.0, form=form))
    for rep in range(3):
        nrhs = int(rng.integers(1, 8))
        V = rng.standard_normal((nrhs, n)) if nrhs > 1 or rng.random() < 0.5 else rng.standard_normal(n)
        out = np.empty_like(V)
        plan.kmvm_host(V, out)
        dev = plan.kmvm(torch.from_numpy(V).cuda()).cpu().numpy()
        if not np.array_equal(out, dev):
            bad += 1
            print(f"FAIL case {it}/{rep}: d={d} n={n} nrhs={nrhs} max diff {np.max(np.abs(out - dev))}", flush=True)
    plan.close()
print(f"fuzz_host: 180 calls, {bad} failures")
