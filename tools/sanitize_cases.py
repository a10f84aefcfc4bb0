"""Small cases through every kernel path and entry point, for compute-sanitizer runs
(memcheck / racecheck / synccheck): `bash tools/gpu/run.sh sanitize <tool>`.

Covers the d = 1 single-chunk kernel (user / rank order, 1 and 3 columns, the CG
epilogue), the three-launch d = 1 path, d = 2 / d = 3 level passes (L1 and product,
nu up to 7/2, the lengthscale gradient), K_zx and gp_predict (with its cache), CG (fused
and graph-replayed, GLS, X / beta_OLS), the pivoted-Cholesky preconditioner (create, solve
with 1, 5 and 9 columns, logdet), Algorithm 2 (gp_mbcg), gp_lml and gp_fit."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2508_01864_b200 as g

rng = np.random.default_rng(0)
cases = [(1, 3000, 0, 5), (1, 2500, 0, 3), (2, 3000, 0, 3), (2, 2500, 1, 3), (2, 1500, 1, 7),
         (3, 2100, 0, 5), (3, 1200, 0, 7), (3, 2100, 1, 3), (3, 1300, 1, 5), (2, 1400, 1, 9),
         (3, 1100, 0, 9)]
for d, n, form, two_nu in cases:
    x = torch.from_numpy(rng.random((n, d))).cuda()
    ell = (0.1, 0.2, 0.3)[:d]
    plan = g.Plan(x, g.Kernel(two_nu, ell, form=form))
    V = torch.randn((3, n), dtype=torch.float64, device="cuda")
    plan.kmvm(V)
    plan.kmvm(V[0].contiguous())
    VR = torch.stack([plan.to_rank(V[i].contiguous()) for i in range(3)])
    plan.kmvm_rank(VR)
    plan.kmvm_rank(VR[1].contiguous())
    if d >= 2:
        for s in range(3):
            plan.kmvm_partial(VR, s, 3)
    z = torch.from_numpy(rng.random((300, d))).cuda()
    cr = plan.cross(z)
    cr.kzx(V[0].contiguous())
    cr.close()
    plan.kmvm_dlengthscale(V)   # every (nu, form, d) has a gradient MVM (separated product forms too)
    if d == 1:
        plan.set_option(0, 3)   # the three-launch path
        plan.kmvm(V)
        plan.kmvm_rank(VR[0].contiguous())
        plan.kmvm_dlengthscale(V[1].contiguous())
        plan.set_option(0, 0)
    if form == 1 or d == 1:
        y = torch.randn(n, dtype=torch.float64, device="cuda")
        try:
            a, b, info = plan.cg_solve(y, 0.1, mean=g.MEAN_AFFINE, rtol=1e-6, max_iter=64,
                                       return_x=True, return_ols=True)
            plan.predict(z, a, b)
            plan.predict(z, a, b)   # cached union structure
        except g.GPError:
            pass
    if d == 2 and form == 1 and two_nu == 3:
        y = torch.randn(n, dtype=torch.float64, device="cuda")
        pc = g.Precond(plan, 24)
        pc.factor()
        for nb in (1, 5, 9):
            pc.solve(0.05, torch.randn((nb, n), dtype=torch.float64, device="cuda"))
        pc.logdet(0.05)
        B = torch.randn((4, n), dtype=torch.float64, device="cuda")
        plan.mbcg(B, 0.05, 12, precond=pc)
        plan.mbcg(B, 0.05, 12)
        G = torch.randn((4, n), dtype=torch.float64, device="cuda")
        W = torch.randn((4, 24), dtype=torch.float64, device="cuda")
        plan.lml(y, 0.05, G, W, lanczos_iters=10, cg_rtol=1e-4, precond=pc)
        try:
            plan.cg_solve(y, 0.05, mean=g.MEAN_AFFINE, rtol=1e-6, max_iter=64, precond=pc)
        except g.GPError:
            pass
        pc.close()
        try:
            g.fit(x, g.Kernel(two_nu, ell, form=form), 0.3, y, G, max_steps=2, max_outer=1,
                  lanczos_iters=8, cg_rtol=1e-4)
        except (g.GPError, TypeError):
            pass
    plan.close()
torch.cuda.synchronize()
print("sanitize cases ok")
