"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Dense CPU oracle of the paper's
likelihood machinery, small N only:

  * the log-marginal likelihood and its gradient, exactly (dense Cholesky):
      L = -1/2 r^T A^-1 r - 1/2 log det A - N/2 log 2 pi          PAPER.md L107 [eq gp_log_likelihood]
      dL/dth = 1/2 a^T (dA/dth) a - 1/2 tr(A^-1 dA/dth), a = A^-1 r   L113 [eq gp_log_likelihood_derivative]
    with A = K + sigma^2 I and th in (outputscale s, common lengthscale scale c, sigma):
      dA/ds = 2/s K (L1310 [eq dkernel_dvarsigma]); dA/dlog c = l dK/dl (L1314 [eq dkernel_dl]);
      dA/dsigma = 2 sigma I;
  * Algorithm 2 (L993-1031 [App A, algo MCGLanczos]) -- conjugate gradients with several
    right-hand sides, preconditioner solve s_P, and the Lanczos tridiagonal matrices built
    from the CG coefficients, step by step in the paper's order;
  * the stochastic log-determinant (L1053-1063 [eqn approximationLogDet]):
      log det A ~ N / l sum_i e1^T log(T_i) e1;
  * Hutchinson trace estimates (L1069-1073): tr(A^-1 M) ~ 1/l sum_i z_i^T A^-1 M z_i;
  * the pivoted-Cholesky preconditioner P = L L^T + sigma^2 I (L1076-1078, Harbrecht et al.),
    the Woodbury solve (L1080-1083) and Sylvester's log-determinant (L1087-1095).

Library primitives used as steps: numpy Cholesky / solve / eigh / slogdet.
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as _o

__all__ = [
    "cov_matrix", "dcov_matrices", "lml_exact", "lml_grad_exact", "mbcg", "lanczos_T",
    "slq_logdet", "hutchinson_trace", "pivoted_cholesky", "woodbury_solve",
    "sylvester_logdet", "lml_stochastic", "adam_step", "sigma_update", "alg1_fit",
]


def cov_matrix(x, two_nu, form, ell, outputscale, sigma2):
    """A = K + sigma^2 I, K from the oracle's dense kernel."""
    K = _o.dense_kernel(x, x, two_nu, form, ell, outputscale)
    return K + sigma2 * np.eye(K.shape[0]), K


def dcov_matrices(x, two_nu, form, ell, outputscale, sigma2):
    """dA/ds, dA/dlog c, dA/dsigma for th = (outputscale s, lengthscale scale c, sigma)."""
    K = _o.dense_kernel(x, x, two_nu, form, ell, outputscale)
    dK = _o.dense_dkernel(x, x, two_nu, form, ell, outputscale)
    n = K.shape[0]
    return [2.0 / outputscale * K, dK, 2.0 * math.sqrt(sigma2) * np.eye(n)]


def lml_exact(A, r):
    """eq gp_log_likelihood (L107) by a dense Cholesky factor."""
    C = np.linalg.cholesky(A)
    w = np.linalg.solve(C, r)
    logdet = 2.0 * np.sum(np.log(np.diag(C)))
    quad = float(w @ w)
    n = A.shape[0]
    return -0.5 * quad - 0.5 * logdet - 0.5 * n * math.log(2 * math.pi), quad, logdet


def lml_grad_exact(A, dAs, r):
    """eq gp_log_likelihood_derivative (L113), dense: 1/2 a^T dA a - 1/2 tr(A^-1 dA)."""
    Ainv = np.linalg.inv(A)
    a = Ainv @ r
    return np.array([0.5 * a @ dA @ a - 0.5 * np.trace(Ainv @ dA) for dA in dAs])


def mbcg(fM, B, n_max, tol, X0=None, sP=None):
    """Algorithm 2 (L993-1031) as printed: returns (M_B, n_I, T list, alphas, betas).

    fM: X -> M X (N x l); B: N x l; n_max = bar n_I; tol on ||R||^2 (the whole residual
    matrix, as printed); sP: R -> P^-1 R (identity if None).  T_j are n_max x n_max with the
    leading n_I x n_I block filled; alphas/betas: per-iteration coefficient rows (l each)."""
    B = np.asarray(B, dtype=np.float64)
    if B.ndim == 1:
        B = B[:, None]
    N, l = B.shape
    sP = sP or (lambda R: R.copy())
    MB = np.zeros_like(B) if X0 is None else np.array(X0, dtype=np.float64)
    R = B - fM(MB)                                   # initial residual
    Pb = sP(R)                                       # initial search direction
    k = np.array([Pb[:, j] @ R[:, j] for j in range(l)])
    nI = 0
    T = [np.zeros((n_max, n_max)) for _ in range(l)]
    a_prev = np.ones(l)
    b_prev = np.zeros(l)
    alphas, betas = [], []
    while nI < n_max:
        Tm = fM(Pb)
        alpha = np.array([k[j] / (Pb[:, j] @ Tm[:, j]) for j in range(l)])
        alphas.append(alpha.copy())
        MB = MB + Pb * alpha
        R = R - Tm * alpha
        if np.sum(R * R) < tol:
            return MB, nI, T, np.array(alphas), np.array(betas)
        Z = sP(R)
        k_prev = k
        nI += 1
        k = np.array([Z[:, j] @ R[:, j] for j in range(l)])
        beta = k / k_prev
        betas.append(beta.copy())
        Pb = Z + Pb * beta
        for j in range(l):
            T[j][nI - 1, nI - 1] = 1.0 / alpha[j] + b_prev[j] / a_prev[j]
            if nI < n_max:
                T[j][nI, nI - 1] = T[j][nI - 1, nI] = math.sqrt(beta[j]) / alpha[j]
        a_prev = alpha
        b_prev = beta
    return MB, nI, T, np.array(alphas), np.array(betas)


def lanczos_T(A, z, m):
    """Plain Lanczos tridiagonalisation of A started at z/||z|| with full
    re-orthogonalisation (Saad §6.6; used only to pin the CG-coefficient route)."""
    n = A.shape[0]
    V = np.zeros((n, m))
    a = np.zeros(m)
    b = np.zeros(max(m - 1, 0))
    v = z / np.linalg.norm(z)
    V[:, 0] = v
    w = A @ v
    for j in range(m):
        a[j] = V[:, j] @ w
        w = w - a[j] * V[:, j]
        w = w - V[:, :j + 1] @ (V[:, :j + 1].T @ w)     # re-orthogonalise
        if j + 1 < m:
            b[j] = np.linalg.norm(w)
            V[:, j + 1] = w / b[j]
            w = A @ V[:, j + 1] - b[j] * V[:, j]
    return np.diag(a) + np.diag(b, 1) + np.diag(b, -1)


def slq_logdet(Ts, m_used, N, weights=None):
    """eqn approximationLogDet (L1063): N/l sum_i e1^T log(T_i) e1 on the leading m x m
    blocks; weights (optional) replace N by ||z_i||^2 (the exact Lanczos identity)."""
    l = len(Ts)
    acc = 0.0
    for i, T in enumerate(Ts):
        m = m_used[i] if np.ndim(m_used) else m_used
        lam, U = np.linalg.eigh(T[:m, :m])
        q = float(np.sum(U[0, :] ** 2 * np.log(lam)))
        acc += (weights[i] if weights is not None else N) * q
    return acc / l


def hutchinson_trace(Z, AinvZ, MZ):
    """1/l sum_i z_i^T A^-1 M z_i  (L1069-1073) = 1/l sum_i (A^-1 z_i)^T (M z_i), M, A sym."""
    return float(np.sum(AinvZ * MZ) / Z.shape[1])


def pivoted_cholesky(K, k):
    """Greedy pivoted Cholesky of rank k (Harbrecht et al., cited at L1076): pivot on the
    largest remaining diagonal (ties: smallest index); returns (L N x k, pivots)."""
    n = K.shape[0]
    d = np.diag(K).astype(np.float64).copy()
    L = np.zeros((n, k))
    piv = []
    for i in range(k):
        p = int(np.argmax(d))
        piv.append(p)
        col = K[:, p] - L[:, :i] @ L[p, :i]
        L[:, i] = col / math.sqrt(d[p])
        d = d - L[:, i] ** 2
    return L, np.array(piv)


def woodbury_solve(L, sigma2, y):
    """P^-1 y = y/s^2 - 1/s^4 L (I_k + L^T L / s^2)^-1 L^T y   (L1080-1083)."""
    k = L.shape[1]
    C = np.eye(k) + (L.T @ L) / sigma2
    return y / sigma2 - (L @ np.linalg.solve(C, L.T @ y)) / sigma2 ** 2


def sylvester_logdet(L, sigma2, N):
    """log det(L L^T + s^2 I_N) = 2N log s + log det(I_k + L^T L / s^2)   (L1087-1095)."""
    k = L.shape[1]
    sign, ld = np.linalg.slogdet(np.eye(k) + (L.T @ L) / sigma2)
    return N * math.log(sigma2) + ld


def lml_stochastic(A, dAs, r, Z, m, sP=None, logdet_P=0.0):
    """The paper's estimator with given probes Z (N x l): a = A^-1 r by CG (Alg 2 run to a
    tight tolerance), log det by eqn approximationLogDet on m Lanczos steps of the probes
    (+ log det P when preconditioned, L1085), traces by Hutchinson with the probes' CG
    solutions (L1069-1073).  With a preconditioner the probes are draws of N(0, P)
    (reading R12) and the trace uses tr(A^-1 M) ~ 1/l sum (A^-1 z)^T M (P^-1 z).
    Returns dict(lml, quad, logdet, grad)."""
    N = A.shape[0]
    fM = lambda X: A @ X
    a, _, _, _, _ = mbcg(fM, r[:, None], 4 * N, 1e-30 * float(r @ r), sP=sP)
    a = a[:, 0]
    quad = float(r @ a)
    XZ, nI, T, _, _ = mbcg(fM, Z, m, 0.0, sP=sP)
    logdet = slq_logdet(T, nI, N) + logdet_P
    PZ = Z if sP is None else sP(Z)
    grad = np.array([0.5 * a @ dA @ a - 0.5 * hutchinson_trace(Z, XZ, dA @ PZ) for dA in dAs])
    lml = -0.5 * quad - 0.5 * logdet - 0.5 * N * math.log(2 * math.pi)
    return {"lml": lml, "quad": quad, "logdet": logdet, "grad": grad, "XZ": XZ, "T": T,
            "nI": nI}


# ---------------------------------------------------------------------------
# Algorithm 1: successive gradient descents with the sigma update and
# the GLS / beta-average loop.  GradDescStep is one ADAM step (Kingma & Ba, the optimiser
# the paper uses, L713-714) on theta = (log s, log c) -- c scales every lengthscale --
# ascending the stochastic LML (lml_stochastic with fixed probes).  Reading R13:
# log-parameters, ADAM defaults beta1 = 0.9, beta2 = 0.999, eps = 1e-8, gradNorm =
# ||grad_theta L|| / N.

def adam_step(theta, g, state, lr, b1=0.9, b2=0.999, eps=1e-8):
    """One ADAM ascent step (bias-corrected moments); state = (m, v, t)."""
    m, v, t = state
    t += 1
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    return theta + lr * mh / (np.sqrt(vh) + eps), (m, v, t)


def sigma_update(x, yc, two_nu, form, ell, s, sigma_prev):
    """(sigma)^2 = 1/N y^T (Ktilde + I)^-1 y, Ktilde = K(s / sigma_prev, l)  (Alg 1)."""
    A, _ = cov_matrix(x, two_nu, form, ell, s / sigma_prev, 1.0)
    return math.sqrt(float(yc @ np.linalg.solve(A, yc)) / len(yc))


def alg1_fit(x, y, H, two_nu, form, ell0, s0, sigma0, Z, m, lr=0.05, max_steps=50,
             max_outer=3, grad_tol=1e-4, beta_tol=1e-3, trace=None):
    """Algorithm 1 with the stochastic LML of lml_stochastic (probes Z, m Lanczos steps).
    Returns dict(s, c, sigma, beta, steps, outer)."""
    N = len(y)
    ell0 = np.asarray(ell0, dtype=np.float64)
    beta_ols = _o.ols(H, y)                                  # OLS estimate
    theta = np.array([math.log(s0), 0.0])
    state = (np.zeros(2), np.zeros(2), 0)
    sigma = sigma0
    steps = 0

    def descent(yc):
        nonlocal theta, state, sigma, steps
        while True:
            s, c = math.exp(theta[0]), math.exp(theta[1])
            A, K = cov_matrix(x, two_nu, form, ell0 * c, s, sigma ** 2)
            dK = _o.dense_dkernel(x, x, two_nu, form, ell0 * c, s)
            st = lml_stochastic(A, [2.0 / s * K, dK], yc, Z, m)
            g = np.array([st["grad"][0] * s, st["grad"][1]])  # d/dlog s, d/dlog c
            theta, state = adam_step(theta, g, state, lr)
            steps += 1
            s, c = math.exp(theta[0]), math.exp(theta[1])
            sigma = sigma_update(x, yc, two_nu, form, ell0 * c, s, sigma)
            if trace is not None:
                trace.append((s, c, sigma))
            if np.linalg.norm(g) / N <= grad_tol or steps >= max_steps * (outer + 1):
                return

    outer = 0
    descent(y - H @ beta_ols)                                # descent with OLS-centred y
    beta_avg = np.zeros(H.shape[1])
    beta_old = beta_ols
    beta_gls = beta_ols
    while outer < max_outer:
        s, c = math.exp(theta[0]), math.exp(theta[1])
        A, _ = cov_matrix(x, two_nu, form, ell0 * c, s, sigma ** 2)
        AiH = np.linalg.solve(A, H)
        beta_gls = np.linalg.solve(H.T @ AiH, AiH.T @ y)    # L808-812
        outer += 1
        beta_avg = (outer - 1) / outer * beta_avg + beta_gls / outer
        descent(y - H @ beta_avg)
        change = np.linalg.norm(beta_gls - beta_old)
        beta_old = beta_gls
        if change <= beta_tol:
            break
    return {"s": math.exp(theta[0]), "c": math.exp(theta[1]), "sigma": sigma,
            "beta": beta_gls, "steps": steps, "outer": outer}
