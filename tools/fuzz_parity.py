"""Randomised parity sweep of the apply entry points against the CPU oracle (one-off check,
not part of the test suite): random n, d, nu, form, lengthscales, ties / duplicates, number
of columns, value or lengthscale gradient, user or rank order, K_zx.
    python tools/fuzz_parity.py [cases] [seed]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2508_01864_b200 as g

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
only = int(os.environ.get("FUZZ_ONLY", "-1"))   # re-run one case (same random stream)
bad = 0
for it in range(cases):
    d = int(rng.integers(1, 4))
    nu2 = int(rng.choice([1, 3, 5, 7, 9]))
    form = int(rng.integers(0, 2))
    big = rng.random() < 0.15
    n = int(rng.integers(1, 40000 if big else 5000))
    if d == 1 and rng.random() < 0.3:
        n = int(rng.integers(5000, 300000))
    if d == 1 and rng.random() < 0.08:
        n = int(rng.integers(900_000, 2_400_000))   # the large shapes and the three-launch path
    if d >= 2 and rng.random() < 0.05:
        n = int(rng.integers(40_000, 160_000))
    nrhs = int(rng.choice([1, 1, 2, 5]))
    grad = rng.random() < 0.3
    kzx = (not grad) and rng.random() < 0.2
    rank = (not kzx) and rng.random() < 0.3
    wide = os.environ.get("FUZZ_WIDE") == "1"   # extreme lengthscales, scaled and shifted coordinates
    ell = tuple(float(x) for x in 10 ** (rng.uniform(-3.5, 1.5, d) if wide else rng.uniform(-1.6, 0.2, d)))
    os_ = float(rng.uniform(0.5, 2.0))
    x = rng.random((n, d))
    mode = rng.integers(0, 3)
    if mode == 1:   # coarse grid: ties in every coordinate
        x = np.floor(x * 13) / 13
    elif mode == 2 and n > 10:   # duplicates
        idx = rng.integers(0, n, n // 10)
        x[rng.integers(0, n, n // 10)] = x[idx]
    if wide:
        sc = 10 ** rng.uniform(-2, 3)
        x = x * sc + rng.uniform(-1e4, 1e4)
        ell = tuple(e * sc for e in ell)
    V = rng.standard_normal((nrhs, n))
    fname = ["l1", "product"][form]
    if kzx:
        m = int(rng.integers(1, 800))
        z = rng.random((m, d))
    rows = rng.choice(n, min(n, 200), replace=False)
    rng_case = rng.random()
    if only >= 0 and it != only:
        continue
    if only >= 0:
        np.savez("gpurun_out/fuzz_case.npz", x=x, V=V, ell=np.array(ell), os_=os_, nu2=nu2, form=form, d=d)
    try:
        plan = g.Plan(torch.from_numpy(x).cuda(), g.Kernel(nu2, ell, os_, form=form))
        Vd = torch.from_numpy(V).cuda()
        vin = Vd if nrhs > 1 else Vd[0]
        worst = 0.0
        if kzx:
            if m > 3:
                z[:3] = x[:3] if n >= 3 else z[:3]
            cr = plan.cross(torch.from_numpy(z).cuda())
            out = cr.kzx(vin).cpu().numpy().reshape(nrhs, m)
            zr = rng.choice(m, min(m, 100), replace=False)
            for c in range(nrhs):
                ref, ab = oracle.kzx_rows(x, V[c], z, nu2, fname, ell, os_, rows=zr, return_abs=True)
                worst = max(worst, np.max(np.abs(out[c][zr] - ref)) / max(ab.max() * np.abs(V[c]).max(), 1e-300))
            cr.close()
        elif d >= 2 and not grad and rng_case < 0.25:   # sharded partial applies sum to K v
            G = 2 + int(rng_case * 12)
            vr = torch.stack([plan.to_rank(Vd[c].contiguous()) for c in range(nrhs)])
            acc = torch.zeros_like(vr)
            for sh in range(G):
                acc += plan.kmvm_partial(vr if nrhs > 1 else vr[0], sh, G).reshape(nrhs, n)
            out = torch.stack([plan.from_rank(acc[c].contiguous()) for c in range(nrhs)]).cpu().numpy()
            for c in range(nrhs):
                ref, ab = oracle.kmvm_rows(x, V[c], nu2, fname, ell, os_, rows=rows, return_abs=True)
                worst = max(worst, np.max(np.abs(out[c][rows] - ref)) / max(ab.max() * np.abs(V[c]).max(), 1e-300))
        else:
            if rank:
                vr = torch.stack([plan.to_rank(Vd[c].contiguous()) for c in range(nrhs)])
                vr = vr if nrhs > 1 else vr[0]
                o = plan.kmvm_dlengthscale(vr, rank_order=True) if grad else plan.kmvm_rank(vr)
                o = o.reshape(nrhs, n)
                out = torch.stack([plan.from_rank(o[c].contiguous()) for c in range(nrhs)]).cpu().numpy()
            else:
                o = plan.kmvm_dlengthscale(vin) if grad else plan.kmvm(vin)
                out = o.cpu().numpy().reshape(nrhs, n)
            for c in range(nrhs):
                f = oracle.dkmvm_rows if grad else oracle.kmvm_rows
                ref, ab = f(x, V[c], nu2, fname, ell, os_, rows=rows, return_abs=True)
                worst = max(worst, np.max(np.abs(out[c][rows] - ref)) / max(ab.max() * np.abs(V[c]).max(), 1e-300))
        plan.close()
        ok = worst <= 1e-9
    except Exception as e:   # noqa: BLE001
        ok, worst = False, repr(e)
    if not ok:
        bad += 1
        print(f"FAIL case {it}: d={d} nu={nu2}/2 form={fname} n={n} nrhs={nrhs} grad={grad} kzx={kzx} "
              f"rank={rank} mode={mode} ell={ell}: {worst}", flush=True)
    elif it % 25 == 0:
        print(f"case {it}: d={d} nu={nu2}/2 {fname} n={n} nrhs={nrhs} grad={grad} kzx={kzx} rank={rank}: "
              f"{worst:.1e}", flush=True)
print(f"fuzz: {cases} cases, {bad} failures")
