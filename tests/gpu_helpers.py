"""Shared helpers for the GPU parity tests (test infrastructure)."""
import numpy as np

import oracle

FORM = {0: "l1", 1: "product"}
TOL = 1e-9      # north_star: max|d| <= 1e-9 ||K||_inf ||v||_inf per MVM


def to_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def check_rows(got, x, v, two_nu, form, ell, os_, rows=None, z=None, tol=TOL, what="",
               grad=False):
    """Compare GPU output rows with the oracle; return (maxerr, bound).
    grad: the lengthscale-gradient MVM (l dK/dl) v, bounded by its own ||.||_inf."""
    got = np.asarray(got)
    if grad:
        ref, ab = oracle.dkmvm_rows(x, v, two_nu, form, ell, os_, rows=rows, return_abs=True)
    elif z is None:
        ref, ab = oracle.kmvm_rows(x, v, two_nu, form, ell, os_, rows=rows, return_abs=True)
    else:
        ref, ab = oracle.kzx_rows(x, v, z, two_nu, form, ell, os_, rows=rows, return_abs=True)
    g = got if rows is None else got[rows]
    err = float(np.max(np.abs(g - ref))) if ref.size else 0.0
    bound = tol * float(np.max(ab) if ab.size else 0.0) * float(np.max(np.abs(v)) if v.size else 0.0)
    assert err <= bound, f"{what}: max|d| = {err:.3e} > {bound:.3e}"
    return err, bound
