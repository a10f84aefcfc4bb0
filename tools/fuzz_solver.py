"""Randomised sweep of the solver entry points (CG + GLS + posterior mean, with and without the
pivoted-Cholesky preconditioner) against the dense oracle on small problems (one-off check).
    python tools/fuzz_solver.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2508_01864_b200 as g

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for it in range(cases):
    d = int(rng.integers(1, 4))
    nu2 = int(rng.choice([1, 3, 5, 7]))
    form = 1 if d > 1 and nu2 > 1 else int(rng.integers(0, 2))   # PD kernels only (R4)
    n = int(rng.integers(50, 1400))
    m = int(rng.integers(1, 300))
    ell = tuple(float(v) for v in 10 ** rng.uniform(-1.3, -0.3, d))
    os_ = float(rng.uniform(0.7, 1.5))
    s2 = float(10 ** rng.uniform(-3, -1))
    mean = [g.MEAN_NONE, g.MEAN_AFFINE][int(rng.integers(0, 2))]
    use_pc = rng.random() < 0.4
    x = rng.random((n, d)); z = rng.random((m, d))
    y = np.sin(4 * x[:, 0]) + 0.3 * x.sum(1) + 0.1 * rng.standard_normal(n)
    fname = ["l1", "product"][form]
    try:
        ref = oracle.gp_dense(x, y, z, nu2, fname, ell, os_, s2, mean="none" if mean == g.MEAN_NONE else "affine")
        plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu2, ell, os_, form=form))
        kw = {}
        if use_pc:
            pc = g.Precond(plan, int(rng.integers(4, min(60, n))))
            kw["precond"] = pc
        alpha, beta, info = plan.cg_solve(torch.from_numpy(y).cuda(), s2, mean=mean, rtol=1e-11,
                                          max_iter=20000, **kw)
        mu = plan.predict(torch.from_numpy(z).cuda(), alpha, beta if mean != g.MEAN_NONE else None).cpu().numpy()
        ea = np.max(np.abs(alpha.cpu().numpy() - ref["alpha"])) / (np.linalg.norm(y) / s2)
        em = np.max(np.abs(mu - ref["mu"])) / max(np.abs(ref["mu"]).max(), 1e-300)
        eb = np.max(np.abs(np.array(beta) - ref["beta"])) if mean != g.MEAN_NONE else 0.0
        ok = ea <= 1e-8 and em <= 1e-6 and eb <= 1e-5 and info["relres_max"] <= 1e-11
        msg = f"alpha {ea:.1e} mu {em:.1e} beta {eb:.1e} relres {info['relres_max']:.1e} iters {info['iters']}"
        if use_pc:
            pc.close()
        plan.close()
    except Exception as e:   # noqa: BLE001
        ok, msg = False, repr(e)
    if not ok:
        bad += 1
    if not ok or it % 10 == 0:
        print(f"{'FAIL' if not ok else 'case'} {it}: d={d} nu={nu2}/2 {fname} n={n} m={m} s2={s2:.1e} mean={mean} pc={use_pc}: {msg}",
              flush=True)
print(f"fuzz_solver: {cases} cases, {bad} failures")
