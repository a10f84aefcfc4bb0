"""Randomised sweep of gp_lml (value, log-det, gradients) against the oracle's estimator with the
same probes, in the numerically stable regime (short lengthscales), all kernels incl. the
separated product forms.  One-off check."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle
from oracle import lml as ol
import paper_2508_01864_b200 as g
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for it in range(N):
    d = int(rng.integers(1, 4)); nu2 = int(rng.choice([1, 3, 5, 7, 9]))
    form = 1 if (d > 1 and nu2 > 1) else int(rng.integers(0, 2))
    fname = ["l1", "product"][form]
    n = int(rng.integers(150, 500))
    base = {1: 0.01, 2: 0.05, 3: 0.1}[d]
    ell = [float(base * rng.uniform(0.7, 1.5)) for _ in range(d)]
    s2 = float(rng.uniform(0.03, 0.3)); os_ = float(rng.uniform(0.8, 1.4))
    x = rng.random((n, d))
    ro = np.argsort(x[:, 0], kind="stable")
    try:
        plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu2, tuple(ell), os_, form=form))
        A, K = ol.cov_matrix(x[ro], nu2, fname, ell, os_, s2)
        r = rng.standard_normal(n); G = rng.standard_normal((6, n)); m = 15
        got = plan.lml(torch.from_numpy(r).cuda(), s2, torch.from_numpy(G).cuda(), lanczos_iters=m, cg_rtol=1e-12)
        dAs = [2.0 / os_ * (A - s2 * np.eye(n)), oracle.dense_dkernel(x[ro], x[ro], nu2, fname, ell, os_),
               2.0 * math.sqrt(s2) * np.eye(n)]
        ref = ol.lml_stochastic(A, dAs, r[ro], G[:, ro].T, m)
        errs = [abs(got["lml"] - ref["lml"]) / abs(ref["lml"]), abs(got["logdet"] - ref["logdet"]) / max(abs(ref["logdet"]), 1)]
        errs += [abs(got["grad"][i] - ref["grad"][i]) / max(abs(ref["grad"][i]), 1.0) for i in range(3)]
        ok = max(errs) <= 1e-5
        msg = " ".join(f"{e:.1e}" for e in errs)
        plan.close()
    except Exception as e:   # noqa: BLE001
        ok, msg = False, repr(e)
    if not ok:
        bad += 1
    if not ok or it % 5 == 0:
        print(f"{'FAIL' if not ok else 'case'} {it}: d={d} nu={nu2}/2 {fname} n={n} ell={[round(e, 3) for e in ell]} s2={s2:.2f}: {msg}", flush=True)
print(f"fuzz_lml: {N} cases, {bad} failures")
