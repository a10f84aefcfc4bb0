"""TEST INFRASTRUCTURE ONLY.  Python side of the oracle (see oracle/__init__.py).

Every function restates a definition of the paper; none of them sorts, scans or
decomposes the kernel.  Parity status of each function is pinned in
tests/test_oracle.py (none is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

__all__ = [
    "build_oracle", "kernel_value", "dkernel_value", "kmvm_rows", "dkmvm_rows", "dkzx_rows", "kzx_rows", "dense_kernel",
    "ols", "gp_dense", "max_threads", "FORMS", "dense_dkernel",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "matern_oracle.c")
_LIB = os.path.join(_HERE, "libmatern_oracle.so")
FORMS = {"l1": 0, "product": 1}
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile the C oracle with gcc -O2 -fopenmp (no fast-math: IEEE exp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        dp = ctypes.POINTER(ctypes.c_double)
        lp = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_kernel_value.restype = ctypes.c_double
        lib.oracle_kernel_value.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                                            ctypes.c_double, dp, dp]
        lib.oracle_cross_mvm.restype = None
        lib.oracle_cross_mvm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                                         ctypes.c_double, dp, dp, ctypes.c_int64, dp, lp,
                                         ctypes.c_int64, dp, dp, ctypes.c_int]
        lib.oracle_dkernel_value.restype = ctypes.c_double
        lib.oracle_dkernel_value.argtypes = lib.oracle_kernel_value.argtypes
        lib.oracle_cross_dmvm.restype = None
        lib.oracle_cross_dmvm.argtypes = lib.oracle_cross_mvm.argtypes
        lib.oracle_dense.restype = None
        lib.oracle_dense.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp,
                                     ctypes.c_double, dp, ctypes.c_int64, dp, ctypes.c_int64,
                                     dp, ctypes.c_int]
        lib.oracle_dense_d.restype = None
        lib.oracle_dense_d.argtypes = lib.oracle_dense.argtypes
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a, ndim=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if ndim == 2 and a.ndim == 1:
        a = a.reshape(-1, 1)
    return a


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def kernel_value(two_nu: int, form: str, ell, outputscale: float, a, b) -> float:
    """Ktilde(a, b), PAPER.md L1253 [eq scaled_matern] with L1273-1275 profiles."""
    a = _f64(np.atleast_1d(a)); b = _f64(np.atleast_1d(b)); ell = _f64(np.atleast_1d(ell))
    return float(_load().oracle_kernel_value(two_nu, FORMS[form], a.size, _dp(ell),
                                             outputscale, _dp(a), _dp(b)))


def dkernel_value(two_nu: int, form: str, ell, outputscale: float, a, b) -> float:
    """l dKtilde/dl, every l_k scaled together: L1 -s^2 r k'(r); product: the product rule
    (PAPER.md L1314 [eq dkernel_dl] times l, with the L1320-1322 derivative profiles)."""
    a = _f64(np.atleast_1d(a)); b = _f64(np.atleast_1d(b)); ell = _f64(np.atleast_1d(ell))
    return float(_load().oracle_dkernel_value(two_nu, FORMS[form], a.size, _dp(ell),
                                              outputscale, _dp(a), _dp(b)))


def dkzx_rows(x, v, z, two_nu: int, form: str, ell, outputscale: float = 1.0, rows=None,
              nthreads: int = 0, return_abs: bool = False):
    """(l dK_zx/dl v)_q = sum_i v_i l dKtilde(x_i, z_q)/dl for q in rows."""
    return kzx_rows(x, v, z, two_nu, form, ell, outputscale, rows, nthreads, return_abs,
                    _kind=1)


def dkmvm_rows(x, v, two_nu: int, form: str, ell, outputscale: float = 1.0, rows=None,
               nthreads: int = 0, return_abs: bool = False):
    """(l dK/dl v)_j, the lengthscale-gradient MVM (PAPER.md L1301-1314 [§ Derivative of
    Matern covariance functions]) used by gradient-based hyperparameter fitting."""
    return dkzx_rows(x, v, x, two_nu, form, ell, outputscale, rows, nthreads, return_abs)


def kzx_rows(x, v, z, two_nu: int, form: str, ell, outputscale: float = 1.0, rows=None,
             nthreads: int = 0, return_abs: bool = False, _kind: int = 0):
    """(K_zx v)_q = sum_i v_i Ktilde(x_i, z_q) for q in rows (all if None).

    PAPER.md L92 [k_z], L256 [eq kde].  x: N x d sources, z: M x d targets.
    Returns out (and the absolute row sums, i.e. the rows of ||K||_inf)."""
    x = _f64(x, 2); z = _f64(z, 2); v = _f64(v).ravel(); ell = _f64(np.atleast_1d(ell))
    d = x.shape[1]
    assert z.shape[1] == d and v.size == x.shape[0] and ell.size == d
    if rows is None:
        nrows = z.shape[0]; rp = None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64); nrows = rows.size
        rp = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    out = np.empty(nrows); ab = np.empty(nrows)
    fn = _load().oracle_cross_dmvm if _kind else _load().oracle_cross_mvm
    fn(two_nu, FORMS[form], d, _dp(ell), float(outputscale), _dp(x), _dp(v), x.shape[0],
       _dp(z), rp, nrows, _dp(out), _dp(ab), int(nthreads))
    return (out, ab) if return_abs else out


def kmvm_rows(x, v, two_nu: int, form: str, ell, outputscale: float = 1.0, rows=None,
              nthreads: int = 0, return_abs: bool = False):
    """(K v)_j = sum_i v_i Ktilde(x_i, x_j), PAPER.md L241-247 [eq Ky], for j in rows."""
    return kzx_rows(x, v, x, two_nu, form, ell, outputscale, rows, nthreads, return_abs)


def dense_kernel(a, b, two_nu: int, form: str, ell, outputscale: float = 1.0, nthreads=0):
    """Dense block [Ktilde(a_i, b_j)] (PAPER.md L219-234 [eq covariance_matrix]); small sizes."""
    a = _f64(a, 2); b = _f64(b, 2); ell = _f64(np.atleast_1d(ell))
    out = np.empty((a.shape[0], b.shape[0]))
    _load().oracle_dense(two_nu, FORMS[form], a.shape[1], _dp(ell), float(outputscale),
                         _dp(a), a.shape[0], _dp(b), b.shape[0], _dp(out), int(nthreads))
    return out


def dense_dkernel(a, b, two_nu: int, form: str, ell, outputscale: float = 1.0, nthreads=0):
    """Dense block [l dKtilde(a_i, b_j)/dl] (PAPER.md L1314 times l); small sizes."""
    a = _f64(a, 2); b = _f64(b, 2); ell = _f64(np.atleast_1d(ell))
    out = np.empty((a.shape[0], b.shape[0]))
    _load().oracle_dense_d(two_nu, FORMS[form], a.shape[1], _dp(ell), float(outputscale),
                           _dp(a), a.shape[0], _dp(b), b.shape[0], _dp(out), int(nthreads))
    return out


def ols(H, y):
    """beta_OLS = (H^T H)^{-1} H^T y  (PAPER.md L829 [Algorithm 1, first line])."""
    H = _f64(H, 2)
    G = H.T @ H
    return np.linalg.solve(G, H.T @ _f64(y).ravel())


def gp_dense(x, y, z, two_nu: int, form: str, ell, outputscale: float, sigma2: float,
             mean: str = "affine", H=None, Hz=None):
    """Dense GP posterior mean with GLS fixed effects, for small N (O(N^3)).

    A = K + sigma^2 I  (PAPER.md L151-153 [eq gp_mean_system])
    beta_GLS = (H^T A^{-1} H)^{-1} H^T A^{-1} y  (PAPER.md L808-812 [§3.2 GLS display])
    alpha = A^{-1} (y - H beta)                  (PAPER.md L86 [eq gp_mean])
    mu(z) = h(z)^T beta + K_zx alpha             (PAPER.md L86, L149 [eq gp_mean_2])
    mean: "none" (m = 0), "affine" (h(x) = [1, x], L73 [eq BetaLin]) or "basis"
    (user H / Hz, L79 [eq BetaFunc]).  A^{-1} is applied through a Cholesky factor
    (library primitive).  Returns dict(alpha, beta, beta_ols, mu, A_inv_y, A_inv_H).
    """
    x = _f64(x, 2); z = _f64(z, 2); y = _f64(y).ravel()
    K = dense_kernel(x, x, two_nu, form, ell, outputscale)
    A = K + sigma2 * np.eye(x.shape[0])
    C = np.linalg.cholesky(A)

    def solve(B):
        return np.linalg.solve(C.T, np.linalg.solve(C, B))

    Ainv_y = solve(y)
    res = {"A_inv_y": Ainv_y}
    if mean == "none":
        beta = np.zeros(0); alpha = Ainv_y; hz = np.zeros((z.shape[0], 0))
        res["beta_ols"] = beta; res["A_inv_H"] = np.zeros((x.shape[0], 0))
    else:
        if mean == "affine":
            Hx = np.hstack([np.ones((x.shape[0], 1)), x])
            hz = np.hstack([np.ones((z.shape[0], 1)), z])
        else:
            Hx = _f64(H, 2); hz = _f64(Hz, 2)
        Ainv_H = solve(Hx)
        beta = np.linalg.solve(Hx.T @ Ainv_H, Hx.T @ Ainv_y)
        alpha = Ainv_y - Ainv_H @ beta
        res["beta_ols"] = ols(Hx, y); res["A_inv_H"] = Ainv_H
    Kzx = dense_kernel(z, x, two_nu, form, ell, outputscale)
    res.update(alpha=alpha, beta=beta, mu=hz @ beta + Kzx @ alpha)
    return res


def timed_kmvm_rows(*args, **kw):
    """kmvm_rows plus wall seconds (used by bench.py's cpu_baseline leg)."""
    t0 = time.perf_counter()
    out = kmvm_rows(*args, **kw)
    return out, time.perf_counter() - t0
