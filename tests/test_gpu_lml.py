"""GPU parity of the likelihood machinery against oracle/lml.py:
pivoted-Cholesky factor, Woodbury solve, Sylvester log-det, Algorithm 2 coefficient
histories, the stochastic LML / gradient with the same probes, preconditioned CG.

Tolerances: the GPU and the oracle run the same recurrences in float64 with different
summation orders (and the GPU's K v differs from the dense product by ~1e-14 relative).
CG / Lanczos coefficients are, depending on the spectrum, either stable or extremely
sensitive to such perturbations once the Krylov basis loses orthogonality (measured with
the oracle alone: a 1e-13 relative perturbation of A moves alpha_25 by up to O(1) for
smooth kernels with long lengthscales, by ~1e-12 for short ones).  Tight 1e-7 checks use
the stable instances (short lengthscales: many comparable eigenvalues); the sensitive
regime is checked against the oracle's own spread under perturbations of A at the MVM
error level.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W
from oracle import lml as ol
from gpu_helpers import to_dev

pytestmark = pytest.mark.gpu


def _rank_order(x):
    return np.argsort(x[:, 0], kind="stable")


def _problem(n, d, seed, two_nu=3, form="l1", ell=None, os_=1.0):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    ell = ell or [0.15, 0.25, 0.3][:d]
    return x, ell, two_nu, form, os_


@pytest.mark.parametrize("d,form", [(1, "l1"), (2, "product"), (2, "l1"), (3, "l1")])
def test_pivoted_cholesky_factor(gpm, d, form):
    x, ell, two_nu, _, os_ = _problem(900, d, 1 + d)
    k = 24
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=0 if form == "l1" else 1))
    pc = gpm.Precond(plan, k)
    piv, L = pc.factor()
    ro = _rank_order(x)                       # the GPU breaks diagonal ties by x1-rank
    K = oracle.dense_kernel(x[ro], x[ro], two_nu, form, ell, os_)
    Lo, po = ol.pivoted_cholesky(K, k)
    assert np.array_equal(piv, ro[po])
    Lu = np.empty((k, 900))
    Lu[:, ro] = Lo.T
    assert np.max(np.abs(L.cpu().numpy() - Lu)) <= 1e-10 * os_ ** 2
    # Woodbury solve and Sylvester log-det
    s2 = 0.07
    r = np.random.default_rng(3).standard_normal((2, 900))
    z = pc.solve(s2, to_dev(r)).cpu().numpy()
    zo = ol.woodbury_solve(Lo, s2, r[:, ro].T).T
    zu = np.empty_like(zo); zu[:, ro] = zo
    assert np.max(np.abs(z - zu)) <= 1e-9 * np.max(np.abs(zu))
    assert pc.logdet(s2) == pytest.approx(ol.sylvester_logdet(Lo, s2, 900), rel=1e-11)
    pc.close()


STABLE = [(1, 3, "l1", [0.01], 0.1), (2, 3, "product", [0.05, 0.05], 0.05),
          (3, 5, "l1", [0.1, 0.1, 0.1], 0.2), (2, 5, "product", [0.04, 0.05], 0.05),
          (3, 3, "product", [0.08, 0.1, 0.09], 0.1), (2, 9, "product", [0.04, 0.05], 0.05)]


@pytest.mark.parametrize("case", range(len(STABLE)))
@pytest.mark.parametrize("precond", [False, True])
def test_mbcg_coefficients_and_solutions(gpm, case, precond):
    d, two_nu, form, ell, s2 = STABLE[case]
    x, ell, two_nu, form, os_ = _problem(700, d, 5 + d, two_nu=two_nu, form=form, ell=ell)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=0 if form == "l1" else 1))
    ro = _rank_order(x)
    A, K = ol.cov_matrix(x[ro], two_nu, form, ell, os_, s2)
    B = np.random.default_rng(6).standard_normal((3, 700))
    m = 25
    pc, sP = None, None
    if precond:
        pc = gpm.Precond(plan, 12)
        Lo, _ = ol.pivoted_cholesky(K, 12)
        sP = lambda R: ol.woodbury_solve(Lo, s2, R)
    X, ah, bh, it = plan.mbcg(to_dev(B), s2, m, 0.0, precond=pc)
    Xo, nI, T, alo, beo = ol.mbcg(lambda V: A @ V, B[:, ro].T, m, 0.0, sP=sP)
    assert it == [m] * 3 and nI == m
    assert np.allclose(ah, alo, rtol=1e-7, atol=0)
    assert np.allclose(bh[:m - 1], beo[:m - 1], rtol=1e-7, atol=0)
    Xu = np.empty((3, 700)); Xu[:, ro] = Xo.T
    assert np.max(np.abs(X.cpu().numpy() - Xu)) <= 1e-7 * np.max(np.abs(Xu))
    if pc:
        pc.close()


def test_mbcg_rtol_stops_and_solves(gpm):
    x, ell, two_nu, form, os_ = _problem(1500, 1, 8, two_nu=3)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_))
    b = np.random.default_rng(9).standard_normal(1500)
    X, ah, bh, it = plan.mbcg(to_dev(b), 0.05, 2000, 1e-10)
    assert it[0] < 2000
    Kx = oracle.kmvm_rows(x, X.cpu().numpy()[0], two_nu, "l1", ell, os_)
    res = b - Kx - 0.05 * X.cpu().numpy()[0]
    assert np.linalg.norm(res) <= 2e-9 * np.linalg.norm(b)


@pytest.mark.parametrize("case", range(len(STABLE)))
@pytest.mark.parametrize("precond", [False, True])
def test_lml_matches_oracle_estimator(gpm, case, precond):
    d, two_nu, form, ell, s2 = STABLE[case]
    x, ell, _, _, _ = _problem(600, d, 20 + d, two_nu=two_nu, form=form, ell=ell)
    os_ = 1.3
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=0 if form == "l1" else 1))
    ro = _rank_order(x)
    A, K = ol.cov_matrix(x[ro], two_nu, form, ell, os_, s2)
    rng = np.random.default_rng(30 + d)
    r = rng.standard_normal(600)
    G = rng.standard_normal((8, 600))
    m = 20
    kw, sP, ldP = {}, None, 0.0
    Z = G[:, ro].T
    if precond:
        kk = 10
        Wn = rng.standard_normal((8, kk))
        pc = gpm.Precond(plan, kk)
        kw = {"precond": pc, "W": to_dev(Wn)}
        Lo, _ = ol.pivoted_cholesky(K, kk)
        sP = lambda R: ol.woodbury_solve(Lo, s2, R)
        ldP = ol.sylvester_logdet(Lo, s2, 600)
        Z = Lo @ Wn.T + math.sqrt(s2) * G[:, ro].T
    got = plan.lml(to_dev(r), s2, to_dev(G), lanczos_iters=m, cg_rtol=1e-12, **kw)
    has_dl = True   # every (nu, form, d) has a lengthscale-gradient MVM
    dAs = [2.0 / os_ * (A - s2 * np.eye(600)),
           oracle.dense_dkernel(x[ro], x[ro], two_nu, form, ell, os_) if has_dl
           else np.zeros((600, 600)),
           2.0 * math.sqrt(s2) * np.eye(600)]
    ref = ol.lml_stochastic(A, dAs, r[ro], Z, m, sP=sP, logdet_P=ldP)
    assert got["quad"] == pytest.approx(ref["quad"], rel=1e-9)
    assert got["logdet"] == pytest.approx(ref["logdet"], rel=1e-7, abs=1e-7)
    assert got["lml"] == pytest.approx(ref["lml"], rel=1e-7)
    assert got["lanczos_iters"] == m
    assert got["grad"][0] == pytest.approx(ref["grad"][0], rel=1e-6, abs=1e-6)
    assert got["grad"][2] == pytest.approx(ref["grad"][2], rel=1e-6, abs=1e-6)
    if has_dl:
        assert got["grad"][1] == pytest.approx(ref["grad"][1], rel=1e-6, abs=1e-6)
    else:
        assert math.isnan(got["grad"][1])


def test_lml_sensitive_regime_within_oracle_spread(gpm):
    """Long lengthscale, smooth kernel: Lanczos coefficients are ill-determined in float64;
    the GPU log-det must lie within 10x the oracle's own spread under 1e-12-relative
    symmetric perturbations of A (plus 1e-9 relative)."""
    x, ell, two_nu, form, os_ = _problem(600, 2, 77, two_nu=5, form="product", ell=[0.15, 0.25])
    s2 = 0.1
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=1))
    ro = _rank_order(x)
    A, K = ol.cov_matrix(x[ro], two_nu, form, ell, os_, s2)
    rng = np.random.default_rng(78)
    r = rng.standard_normal(600)
    G = rng.standard_normal((8, 600))
    got = plan.lml(to_dev(r), s2, to_dev(G), lanczos_iters=20, cg_rtol=1e-12)
    refs = []
    for k in range(3):
        E = rng.standard_normal(A.shape)
        E = (E + E.T) * (1e-12 * np.abs(A).max() if k else 0.0)
        _, nI, T, _, _ = ol.mbcg(lambda V: (A + E) @ V, G[:, ro].T, 20, 0.0)
        refs.append(ol.slq_logdet(T, nI, 600))
    spread = max(refs) - min(refs)
    assert abs(got["logdet"] - refs[0]) <= 10 * spread + 1e-9 * abs(refs[0])


def test_lml_close_to_exact(gpm):
    """With 64 probes and 40 Lanczos steps the estimate sits near the dense LML."""
    x, ell, two_nu, form, os_ = _problem(800, 1, 41, two_nu=3)
    s2 = 0.1
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_))
    A, K = ol.cov_matrix(x, two_nu, "l1", ell, os_, s2)
    rng = np.random.default_rng(42)
    r = rng.standard_normal(800)
    got = plan.lml(to_dev(r), s2, to_dev(rng.standard_normal((64, 800))), lanczos_iters=40)
    ex, quad, logdet = ol.lml_exact(A, r)
    assert got["quad"] == pytest.approx(quad, rel=1e-7)
    assert abs(got["logdet"] - logdet) <= 0.02 * abs(logdet)


def test_preconditioned_cg_solve(gpm):
    c = W.scaled(W.CONFIGS[5], 3000, m=200)
    x = W.config_points(c); y = W.config_response(c, x); z = W.config_queries(c)
    s2 = c.noise_sigma ** 2
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, c.ell, form=1))
    a0, b0, i0 = plan.cg_solve(to_dev(y), s2, mean=gpm.MEAN_AFFINE, rtol=1e-10)
    pc = gpm.Precond(plan, 150)
    a1, b1, i1 = plan.cg_solve(to_dev(y), s2, mean=gpm.MEAN_AFFINE, rtol=1e-10, precond=pc)
    assert i1["relres_max"] <= 1e-10 and i1["iters"] < i0["iters"] / 2
    ref = oracle.gp_dense(x, y, z, 3, "product", c.ell, 1.0, s2, mean="affine")
    assert np.allclose(b1, ref["beta"], atol=1e-6)
    assert np.max(np.abs(a1.cpu().numpy() - ref["alpha"])) <= 1e-10 * np.linalg.norm(y) / s2 * 10
    assert np.max(np.abs(a1.cpu().numpy() - a0.cpu().numpy())) <= 1e-9 * np.linalg.norm(y) / s2 * 10
    pc.close()


def test_lml_errors(gpm):
    x = np.random.default_rng(0).random((200, 1))
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1,)))
    pc = gpm.Precond(plan, 5)
    G = to_dev(np.ones((2, 200)))
    with pytest.raises(ValueError):
        plan.lml(to_dev(np.ones(200)), 0.1, G, precond=pc)          # W missing
    with pytest.raises(gpm.GPError) as e:
        gpm.Precond(plan, 2000)
    assert e.value.name == "INVALID_ARG"
    other = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1,)))
    with pytest.raises(gpm.GPError):
        other.cg_solve(to_dev(np.ones(200)), 0.1, precond=pc)


@pytest.mark.parametrize("d,two_nu,form", [(1, 3, "l1"), (2, 1, "l1"), (2, 3, "product"),
                                             (2, 5, "product"), (3, 3, "product")])
def test_fit_alg1_matches_oracle_trajectory(gpm, d, two_nu, form):
    """Algorithm 1 with the same probes: a few ADAM steps, one GLS round -- the GPU and the
    oracle follow the same trajectory (gradients agree to ~1e-7, ADAM is smooth in them)."""
    rng = np.random.default_rng(60 + d)
    n = 400
    x = rng.random((n, d))
    H = np.hstack([np.ones((n, 1)), x])
    y = H @ np.array([1.0, 0.5, -0.3, 0.2][:1 + d]) + np.sin(5 * x[:, 0]) + 0.2 * rng.standard_normal(n)
    G = rng.standard_normal((8, n))
    ell0 = [0.02, 0.2][:d] if d == 1 else [0.05] * d
    ro = _rank_order(x)
    kw = dict(lr=0.05, max_steps=4, max_outer=1, grad_tol=1e-300, beta_tol=1e-300,
              lanczos_iters=20, cg_rtol=1e-12)
    got = gpm.fit(to_dev(x), gpm.Kernel(two_nu, tuple(ell0), 0.8, form=0 if form == "l1" else 1),
                  0.5, to_dev(y), to_dev(G), **kw)
    ref = ol.alg1_fit(x[ro], y[ro], H[ro], two_nu, form, ell0, 0.8, 0.5, G[:, ro].T, 20,
                      lr=0.05, max_steps=4, max_outer=1, grad_tol=1e-300, beta_tol=1e-300)
    assert got["steps"] == ref["steps"] == 8 and got["outer"] == ref["outer"] == 1
    assert got["kernel"].outputscale == pytest.approx(ref["s"], rel=1e-6)
    assert got["kernel"].lengthscale[0] == pytest.approx(ell0[0] * ref["c"], rel=1e-6)
    assert got["sigma"] == pytest.approx(ref["sigma"], rel=1e-6)
    assert np.allclose(got["beta"], ref["beta"], rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("nb", [1, 2, 3, 4, 5, 8, 9])
def test_woodbury_streaming_kernels(gpm, nb, monkeypatch):
    """P^-1 R by the streaming L^T R / L Y kernels (nb <= 8; nb = 9 takes the cuBLAS GEMMs)
    vs the oracle's Woodbury solve, with n spanning several 1024-row blocks and a ragged
    tail; and equal to the cuBLAS path to rounding (GPM_WOODBURY_CUBLAS)."""
    n, k, s2 = 5000 + 37, 40, 0.05
    x, ell, two_nu, _, os_ = _problem(n, 2, 400 + nb, ell=[0.1, 0.2])
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=1))
    pc = gpm.Precond(plan, k)
    _, L = pc.factor()
    Lu = L.cpu().numpy().T                    # user order, n x k: P = L L^T + s2 I
    r = np.random.default_rng(nb).standard_normal((nb, n))
    z = pc.solve(s2, to_dev(r)).cpu().numpy()
    zo = ol.woodbury_solve(Lu, s2, r.T).T
    assert np.max(np.abs(z - zo)) <= 1e-9 * np.max(np.abs(zo))
    monkeypatch.setenv("GPM_WOODBURY_CUBLAS", "1")
    zc = pc.solve(s2, to_dev(r)).cpu().numpy()
    assert np.max(np.abs(z - zc)) <= 1e-12 * np.max(np.abs(zc))
    pc.close()


def test_solver_entry_points_do_not_leak_device_memory(gpm):
    """Repeated gp_precond_solve / gp_mbcg / preconditioned CG calls return their scratch:
    free device memory is unchanged after 10 more rounds (library buffers are owning)."""
    import torch
    n = 20000
    x, ell, two_nu, _, os_ = _problem(n, 2, 900, ell=[0.1, 0.2])
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=1))
    pc = gpm.Precond(plan, 20)
    r = to_dev(np.random.default_rng(1).standard_normal((3, n)))
    y = to_dev(np.random.default_rng(2).standard_normal(n))

    def one_round():
        pc.solve(0.05, r)
        plan.mbcg(r, 0.05, 30, 0.0)
        plan.cg_solve(y, 0.05, mean=gpm.MEAN_AFFINE, rtol=1e-8, max_iter=5000, precond=pc)
        torch.cuda.synchronize()

    one_round()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(10):
        one_round()
    assert torch.cuda.mem_get_info()[0] >= free0 - (4 << 20)
    pc.close()


def test_woodbury_streaming_rank768_five_columns(gpm):
    """k_wly's dynamic Y (8 k NB bytes) plus its static partials crosses 48 KB at
    k = 761..768 with NB = 8 (5..8 columns): the launch must opt in to the larger carve-out."""
    n, k, s2 = 3000, 768, 0.05
    x, ell, two_nu, _, os_ = _problem(n, 2, 777, ell=[0.1, 0.2])
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=1))
    pc = gpm.Precond(plan, k)
    _, L = pc.factor()
    Lu = L.cpu().numpy().T
    r = np.random.default_rng(5).standard_normal((5, n))
    z = pc.solve(s2, to_dev(r)).cpu().numpy()
    zo = ol.woodbury_solve(Lu, s2, r.T).T
    assert np.max(np.abs(z - zo)) <= 1e-8 * np.max(np.abs(zo))
    pc.close()
    plan.close()


def test_plan_destroyed_before_its_preconditioner(gpm):
    """gp_destroy while a preconditioner is alive defers the free; the
    preconditioner stays usable and frees the plan with itself."""
    n = 2000
    x, ell, two_nu, _, os_ = _problem(n, 2, 778, ell=[0.1, 0.2])
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, tuple(ell), os_, form=1))
    pc = gpm.Precond(plan, 16)
    r = np.random.default_rng(6).standard_normal((2, n))
    z0 = pc.solve(0.1, to_dev(r)).cpu().numpy()
    plan.close()
    z1 = pc.solve(0.1, to_dev(r)).cpu().numpy()
    assert np.array_equal(z0, z1)
    pc.close()
