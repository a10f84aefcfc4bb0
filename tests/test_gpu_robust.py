"""Robustness of the CUDA path at the edges of the input space, against the oracle on all
rows: coordinates far from the origin (catastrophic-cancellation risk in the gaps), very
short lengthscales (K ~ diagonal, e^{-gap} underflows to 0) and very long ones (K ~ a
constant matrix, every pair contributes), in every d = 1 path and for d = 2, 3."""
import numpy as np
import pytest

from gpu_helpers import check_rows, to_dev

pytestmark = pytest.mark.gpu


def _x(kind, n, d, seed):
    rng = np.random.default_rng(seed)
    if kind == "offset":
        return 1.0e4 + rng.random((n, d))
    if kind == "wide":
        return rng.standard_normal((n, d)) * 1.0e3
    return rng.random((n, d))


@pytest.mark.parametrize("path", [0, 3])
@pytest.mark.parametrize("kind,ell", [("offset", 0.05), ("wide", 1.0), ("unit", 1e-5),
                                      ("unit", 1e3), ("offset", 1e3)])
@pytest.mark.parametrize("two_nu", [1, 5])
def test_d1_edges(gpm, path, kind, ell, two_nu):
    n = 5000
    x = _x(kind, n, 1, n + two_nu)
    v = np.random.default_rng(1).standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, (ell,)))
    if path:
        plan.set_option(0, path)
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "l1", (ell,), 1.0, what=f"d1 {kind} ell={ell} path={path}")
    plan.close()


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("kind,ell", [("offset", 0.1), ("unit", 1e-5), ("unit", 1e3)])
def test_d23_edges(gpm, d, kind, ell):
    n = 3000
    x = _x(kind, n, d, 10 * d)
    v = np.random.default_rng(2).standard_normal(n)
    ells = (ell,) * d
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3 if d == 2 else 5, ells))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, 3 if d == 2 else 5, "l1", ells, 1.0, what=f"d{d} {kind} ell={ell}")
    plan.close()


@pytest.mark.parametrize("d,two_nu,form", [(1, 7, 0), (2, 9, 1), (3, 5, 0), (3, 3, 1)])
def test_far_offset_short_lengthscale(gpm, d, two_nu, form):
    """Coordinates 1e4 from the origin with lengthscales of 1e-5..1e-3 of the data's extent:
    offset / l ~ 1e9, so scaling before centring would lose 1e-7 of every scaled distance
    (found by tools/fuzz_parity.py with FUZZ_WIDE=1); the plan centres on the first point."""
    rng = np.random.default_rng(100 + d)
    n = 3000
    x = -9.3e3 + rng.random((n, d))
    ell = tuple(float(e) for e in 10 ** rng.uniform(-4.5, -2.5, d))
    v = rng.standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.0, form=form))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, ["l1", "product"][form], ell, 1.0, what=f"offset d={d}")
    g = plan.kmvm_dlengthscale(to_dev(v)).cpu().numpy()
    check_rows(g, x, v, two_nu, ["l1", "product"][form], ell, 1.0, grad=True, what=f"offset grad d={d}")
    plan.close()
