"""Pins of the likelihood oracle (oracle/lml.py) -- no GPU.

Independent of the oracle's own formulas:
  * Lanczos coefficients from CG (Alg 2) == a plain re-orthogonalised
    Lanczos run (Saad §6.6-6.7);
  * Gauss-Lanczos quadrature is exact once Lanczos terminates: for A with q distinct
    eigenvalues, ||z||^2 e1^T log(T_q) e1 = z^T log(A) z (eigendecomposition of A);
  * Hutchinson with the probes sqrt(N) e_i is the exact trace, so the paper's stochastic
    LML (L1053-1073) equals the dense LML on such matrices;
  * Woodbury / Sylvester (L1080-1095) against dense solves / slogdet;
  * pivoted Cholesky of full rank reproduces K;
  * the dense LML against scipy's multivariate normal log-density, its gradient against
    central finite differences of the LML in (outputscale, lengthscale scale, sigma).
"""
import math

import numpy as np
import pytest
from scipy.stats import multivariate_normal

import oracle
from oracle import lml as ol


def _spd_few_eigs(n, eigs, seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.array([eigs[i % len(eigs)] for i in range(n)], dtype=float)
    return (Q * lam) @ Q.T


def test_cg_lanczos_coefficients_match_plain_lanczos():
    rng = np.random.default_rng(1)
    x = rng.random((80, 2))
    A, _ = ol.cov_matrix(x, 3, "product", [0.3, 0.3], 1.0, 0.5)
    Z = rng.standard_normal((80, 3))
    m = 12
    _, nI, T, _, _ = ol.mbcg(lambda X: A @ X, Z, m, 0.0)
    assert nI == m
    for j in range(3):
        Tl = ol.lanczos_T(A, Z[:, j], m)
        assert np.max(np.abs(T[j] - Tl)) <= 1e-9 * np.max(np.abs(Tl))


def test_mbcg_solves_and_preconditioned_solves():
    rng = np.random.default_rng(2)
    x = rng.random((120, 1))
    A, K = ol.cov_matrix(x, 5, "l1", [0.2], 1.3, 0.05)
    B = rng.standard_normal((120, 2))
    X, _, _, _, _ = ol.mbcg(lambda V: A @ V, B, 600, 1e-24)
    assert np.allclose(A @ X, B, atol=1e-9)
    L, _ = ol.pivoted_cholesky(K, 15)
    sP = lambda R: ol.woodbury_solve(L, 0.05, R)
    Xp, nIp, _, _, _ = ol.mbcg(lambda V: A @ V, B, 600, 1e-24, sP=sP)
    _, nI0, _, _, _ = ol.mbcg(lambda V: A @ V, B, 600, 1e-24)
    assert np.allclose(A @ Xp, B, atol=1e-9)
    assert nIp < nI0                               # the preconditioner helps


def test_lanczos_quadrature_exact_after_termination():
    eigs = [0.3, 1.0, 2.5, 7.0, 11.0]
    A = _spd_few_eigs(40, eigs, 3)
    z = np.random.default_rng(4).standard_normal(40)
    _, nI, T, _, _ = ol.mbcg(lambda X: A @ X, z[:, None], len(eigs), 0.0)
    lam, U = np.linalg.eigh(A)
    exact = float((U.T @ z) ** 2 @ np.log(lam))
    got = ol.slq_logdet(T, nI, 40, weights=[float(z @ z)])
    assert got == pytest.approx(exact, rel=1e-9)


def test_stochastic_lml_equals_dense_with_unit_probes():
    """Probes sqrt(N) e_i: ||z||^2 = N (the paper's approximation becomes exact) and the
    Hutchinson sums are exact traces; q distinct eigenvalues make q Lanczos steps exact."""
    eigs = [0.5, 1.5, 4.0]
    n = 30
    A = _spd_few_eigs(n, eigs, 5)
    rng = np.random.default_rng(6)
    S = rng.standard_normal((n, n))
    dAs = [S + S.T, np.eye(n)]
    r = rng.standard_normal(n)
    Z = math.sqrt(n) * np.eye(n)
    st = ol.lml_stochastic(A, dAs, r, Z, len(eigs))
    ex, quad, logdet = ol.lml_exact(A, r)
    assert st["quad"] == pytest.approx(quad, rel=1e-9)
    assert st["logdet"] == pytest.approx(logdet, rel=1e-9, abs=1e-9)
    assert st["lml"] == pytest.approx(ex, rel=1e-9)
    assert np.allclose(st["grad"], ol.lml_grad_exact(A, dAs, r), rtol=1e-8, atol=1e-9)


def test_woodbury_and_sylvester():
    rng = np.random.default_rng(7)
    L = rng.standard_normal((50, 6))
    s2 = 0.3
    P = L @ L.T + s2 * np.eye(50)
    y = rng.standard_normal((50, 2))
    assert np.allclose(ol.woodbury_solve(L, s2, y), np.linalg.solve(P, y), atol=1e-10)
    assert ol.sylvester_logdet(L, s2, 50) == pytest.approx(np.linalg.slogdet(P)[1], rel=1e-12)


def test_pivoted_cholesky_full_rank_and_greedy_decrease():
    rng = np.random.default_rng(8)
    x = rng.random((40, 2))
    K = oracle.dense_kernel(x, x, 5, "product", [0.4, 0.4], 1.1)
    L, piv = ol.pivoted_cholesky(K, 40)
    assert np.max(np.abs(L @ L.T - K)) <= 1e-8
    assert sorted(piv.tolist()) == list(range(40))
    prev = np.inf
    for k in (1, 5, 10, 20):
        Lk, _ = ol.pivoted_cholesky(K, k)
        res = np.trace(K - Lk @ Lk.T)
        assert res < prev
        prev = res


def test_lml_exact_against_scipy_logpdf():
    rng = np.random.default_rng(9)
    x = rng.random((60, 2))
    A, _ = ol.cov_matrix(x, 3, "product", [0.2, 0.3], 0.8, 0.1)
    r = rng.standard_normal(60)
    ex, _, _ = ol.lml_exact(A, r)
    assert ex == pytest.approx(multivariate_normal(mean=np.zeros(60), cov=A).logpdf(r), rel=1e-10)


@pytest.mark.parametrize("d,two_nu", [(1, 1), (1, 5), (2, 3), (3, 5)])
def test_lml_gradient_against_finite_differences(d, two_nu):
    rng = np.random.default_rng(10 + d)
    x = rng.random((70, d))
    ell = np.array([0.3, 0.4, 0.5][:d])
    s, s2 = 1.2, 0.2
    r = rng.standard_normal(70)

    def L(s_, c_, sig_):
        A, _ = ol.cov_matrix(x, two_nu, "l1", ell * c_, s_, sig_ ** 2)
        return ol.lml_exact(A, r)[0]

    A, _ = ol.cov_matrix(x, two_nu, "l1", ell, s, s2)
    g = ol.lml_grad_exact(A, ol.dcov_matrices(x, two_nu, "l1", ell, s, s2), r)
    h = 1e-5
    sig = math.sqrt(s2)
    fd = [(L(s + h, 1, sig) - L(s - h, 1, sig)) / (2 * h),
          (L(s, math.exp(h), sig) - L(s, math.exp(-h), sig)) / (2 * h),
          (L(s, 1, sig + h) - L(s, 1, sig - h)) / (2 * h)]
    assert np.allclose(g, fd, rtol=1e-6, atol=1e-6)


def test_stochastic_logdet_is_unbiased_within_noise():
    """Gaussian probes (the paper's law): the SLQ estimate lies within 4 standard errors of
    log det A (the probe spread estimates the error)."""
    rng = np.random.default_rng(11)
    x = rng.random((300, 1))
    A, _ = ol.cov_matrix(x, 3, "l1", [0.1], 1.0, 0.1)
    Z = rng.standard_normal((300, 64))
    _, nI, T, _, _ = ol.mbcg(lambda X: A @ X, Z, 40, 0.0)
    per = np.array([ol.slq_logdet([T[j]], nI, 300) for j in range(64)])
    exact = np.linalg.slogdet(A)[1]
    assert abs(per.mean() - exact) <= 4 * per.std() / math.sqrt(64) + 1e-6


def test_preconditioned_stochastic_lml_exact_with_structured_probes():
    """Reading R12: probes z ~ N(0, P).  With z_i = sqrt(N) P^{1/2} e_i (so z z^T / l = P
    exactly) and P^{-1/2} A P^{-1/2} having q distinct eigenvalues, q preconditioned Lanczos
    steps give log det(P^-1 A) exactly, + Sylvester's log det P = log det A, and the
    preconditioned Hutchinson traces are exact."""
    n = 24
    rng = np.random.default_rng(12)
    Lf = rng.standard_normal((n, 4))
    s2 = 0.5
    P = Lf @ Lf.T + s2 * np.eye(n)
    lam, U = np.linalg.eigh(P)
    Ph = (U * np.sqrt(lam)) @ U.T
    M0 = _spd_few_eigs(n, [0.7, 1.3, 3.0], 13)
    A = Ph @ M0 @ Ph
    S = rng.standard_normal((n, n))
    dAs = [S + S.T, np.eye(n)]
    r = rng.standard_normal(n)
    Z = math.sqrt(n) * Ph
    sP = lambda R: ol.woodbury_solve(Lf, s2, R)
    st = ol.lml_stochastic(A, dAs, r, Z, 3, sP=sP, logdet_P=ol.sylvester_logdet(Lf, s2, n))
    ex, quad, logdet = ol.lml_exact(A, r)
    assert st["logdet"] == pytest.approx(logdet, rel=1e-9, abs=1e-9)
    assert st["lml"] == pytest.approx(ex, rel=1e-9)
    assert np.allclose(st["grad"], ol.lml_grad_exact(A, dAs, r), rtol=1e-8, atol=1e-9)


def test_adam_first_step_and_quadratic_convergence():
    """ADAM: the bias-corrected first step moves each coordinate by lr * sign(g); on a
    concave quadratic the iterates converge to the maximiser."""
    th, st = ol.adam_step(np.zeros(2), np.array([3.0, -0.2]), (np.zeros(2), np.zeros(2), 0), 0.1)
    assert np.allclose(th, [0.1, -0.1], atol=1e-7)
    th = np.array([2.0, -1.0]); st = (np.zeros(2), np.zeros(2), 0)
    for _ in range(3000):
        th, st = ol.adam_step(th, -2.0 * (th - np.array([0.5, 0.25])), st, 0.01)
    assert np.allclose(th, [0.5, 0.25], atol=1e-3)


def test_sigma_update_maximises_lml_along_the_ratio():
    """Alg 1's closed form (L846): with s/sigma fixed, sigma^2 = y^T (Ktilde + I)^-1 y / N
    maximises the LML over sigma."""
    rng = np.random.default_rng(14)
    x = rng.random((150, 2)); y = rng.standard_normal(150)
    ell, s, sig0 = [0.2, 0.3], 1.1, 0.4
    sig = ol.sigma_update(x, y, 3, "product", ell, s, sig0)
    ratio = s / sig0

    def L(sg):
        A, _ = ol.cov_matrix(x, 3, "product", ell, ratio * sg, sg ** 2)
        return ol.lml_exact(A, y)[0]
    assert L(sig) >= max(L(sig * 0.98), L(sig * 1.02))


def test_alg1_recovers_simulated_parameters():
    """Data simulated from the model (affine mean + GP + noise, dense Cholesky sampler):
    Alg 1 recovers beta and sigma closely and increases the exact LML."""
    rng = np.random.default_rng(15)
    n = 500
    x = rng.random((n, 2))
    H = np.hstack([np.ones((n, 1)), x])
    beta_true = np.array([1.0, 0.5, -0.3])
    s_true, ell_true, sig_true = 1.0, np.array([0.2, 0.2]), 0.3
    K = oracle.dense_kernel(x, x, 1, "l1", ell_true, s_true)
    f = np.linalg.cholesky(K + 1e-10 * np.eye(n)) @ rng.standard_normal(n)
    y = H @ beta_true + f + sig_true * rng.standard_normal(n)
    Z = rng.standard_normal((n, 16))
    res = ol.alg1_fit(x, y, H, 1, "l1", ell_true * 1.5, 0.7, 0.6, Z, 25, lr=0.05,
                      max_steps=60, max_outer=3)
    assert abs(res["sigma"] - sig_true) < 0.05
    A0, _ = ol.cov_matrix(x, 1, "l1", ell_true * 1.5, 0.7, 0.36)
    A1, _ = ol.cov_matrix(x, 1, "l1", ell_true * 1.5 * res["c"], res["s"], res["sigma"] ** 2)
    # beta within 4 GLS standard errors, cov(beta_GLS) = (H^T A^-1 H)^-1
    se = np.sqrt(np.diag(np.linalg.inv(H.T @ np.linalg.solve(A1, H))))
    assert np.all(np.abs(res["beta"] - beta_true) <= 4 * se)
    r = y - H @ res["beta"]
    assert ol.lml_exact(A1, r)[0] > ol.lml_exact(A0, r)[0]


def _schur_diag(K, sel):
    """diag of the Schur complement K - K[:, S] K[S, S]^-1 K[S, :] (S = sel): the residual
    variance after conditioning on the selected points, computed by a dense solve that
    shares nothing with the pivoted-Cholesky loop."""
    if not sel:
        return np.diag(K).copy()
    S = np.asarray(sel)
    KS = K[:, S]
    return np.diag(K) - np.einsum("ij,ji->i", KS, np.linalg.solve(K[np.ix_(S, S)], KS.T))


def test_pivoted_cholesky_pivot_is_greedy_argmax_of_schur_diagonal():
    """Harbrecht's greedy rule (cited at PAPER.md L1073 [App A.3]): step i pivots on the
    largest diagonal entry of the Schur complement given the earlier pivots (ties: the
    smallest index).  Fails for any other pivot order (e.g. the unpivoted p = i)."""
    rng = np.random.default_rng(21)
    x = rng.random((30, 2))
    K = oracle.dense_kernel(x, x, 3, "product", [0.5, 0.5], 1.0)
    _, piv = ol.pivoted_cholesky(K, 12)
    for i in range(12):
        d = _schur_diag(K, piv[:i].tolist())
        assert d[piv[i]] >= d.max() * (1 - 1e-9), (i, piv[i], int(np.argmax(d)))


def test_pivoted_cholesky_second_pivot_is_farthest_point():
    """1-D, stationary kernel: the diagonal is constant, so the first pivot is index 0
    (tie rule) and the residual variance after it is s^2 (1 - k(r)^2), largest at the
    point farthest from x_0."""
    x = np.array([[0.41], [0.40], [0.05], [0.95], [0.42], [0.60]])
    K = oracle.dense_kernel(x, x, 1, "l1", [0.3], 1.0)
    _, piv = ol.pivoted_cholesky(K, 2)
    assert piv[0] == 0
    assert piv[1] == int(np.argmax(np.abs(x[:, 0] - x[0, 0]))) == 3
