"""GPU parity for nu = 7/2, 9/2: the same
decomposition with p = 3, 4 moments (generic binomial advance / read), L1 form for
d = 1..3; gradients (p + 1 moments) for d = 1, 2 and d = 3 up to nu = 7/2."""
import numpy as np
import pytest

import workloads as W
from gpu_helpers import check_rows, to_dev

pytestmark = pytest.mark.gpu


def _pts(n, d, seed, ties=False):
    rng = np.random.default_rng(seed)
    x = rng.random((n, d))
    if ties:
        x = np.floor(x * 17) / 17
        if n > 4:
            x[n // 2] = x[1]
    return x


@pytest.mark.parametrize("two_nu", [7, 9])
@pytest.mark.parametrize("d,n", [(1, 1), (1, 7), (1, 1000), (1, 7681), (1, 20000), (2, 3),
                                 (2, 2049), (2, 5000), (3, 64), (3, 2049), (3, 5000)])
@pytest.mark.parametrize("grad", [False, True])
def test_high_nu_all_rows(gpm, two_nu, d, n, grad):
    x = _pts(n, d, 31 * n + two_nu + d, ties=(n % 2 == 1))
    v = np.random.default_rng(n + two_nu).standard_normal(n)
    ell = (0.08, 0.2, 0.15)[:d]
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.2, form=0))
    out = (plan.kmvm_dlengthscale(to_dev(v)) if grad else plan.kmvm(to_dev(v))).cpu().numpy()
    check_rows(out, x, v, two_nu, "l1", ell, 1.2, grad=grad,
               what=f"nu={two_nu}/2 d={d} n={n} grad={grad}")


@pytest.mark.parametrize("two_nu", [7, 9])
def test_high_nu_config2_and_multilevel(gpm, two_nu):
    c = W.CONFIGS[2]
    x = W.config_points(c)
    v = W.config_vector(c, 0)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, c.ell))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    rows = W.sample_rows(x, 256)
    check_rows(out, x, v, two_nu, "l1", c.ell, 1.0, rows=rows, what=f"config2 nu={two_nu}/2")
    x3 = _pts(150000, 3, 9 + two_nu)
    v3 = np.random.default_rng(two_nu).standard_normal(150000)
    p3 = gpm.Plan(to_dev(x3), gpm.Kernel(two_nu, (0.1, 0.1, 0.1)))
    o3 = p3.kmvm(to_dev(v3)).cpu().numpy()
    check_rows(o3, x3, v3, two_nu, "l1", (0.1, 0.1, 0.1), 1.0, rows=W.sample_rows(x3, 128),
               what=f"d3 multilevel nu={two_nu}/2")


@pytest.mark.parametrize("two_nu", [7, 9])
@pytest.mark.parametrize("n", [3, 64, 2049, 5000])
@pytest.mark.parametrize("grad", [False, True])
def test_high_nu_product_d2_all_rows(gpm, two_nu, n, grad):
    """d = 2 product form for nu = 7/2, 9/2: (p+1)^2 = 16 / 25 mixed
    moments per channel (wide tile records); the gradient (product rule): (p+2)^2 = 25
    mixed moments for nu = 7/2, the separated two-run form (algebra.cuh SEP 2 / 3) for 9/2."""
    x = _pts(n, 2, 17 * n + two_nu, ties=(n % 2 == 1))
    v = np.random.default_rng(n + two_nu + 3).standard_normal(n)
    ell = (0.1, 0.2)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.1, form=1))
    out = (plan.kmvm_dlengthscale(to_dev(v)) if grad else plan.kmvm(to_dev(v))).cpu().numpy()
    check_rows(out, x, v, two_nu, "product", ell, 1.1, grad=grad,
               what=f"product nu={two_nu}/2 n={n} grad={grad}")


@pytest.mark.parametrize("two_nu", [7, 9])
def test_high_nu_product_d2_multilevel_multirhs(gpm, two_nu):
    """Carried passes (k_cp, k_cp_carry on the wide records) at 2e5 points, 3 columns."""
    n = 200000
    x = _pts(n, 2, 4321 + two_nu)
    V = np.random.default_rng(two_nu).standard_normal((3, n))
    ell = (0.05, 0.08)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.0, form=1))
    out = plan.kmvm(to_dev(V)).cpu().numpy()
    rows = W.sample_rows(x, 128)
    for r in range(3):
        check_rows(out[r], x, V[r], two_nu, "product", ell, 1.0, rows=rows,
                   what=f"product nu={two_nu}/2 multilevel rhs {r}")
    g = plan.kmvm_dlengthscale(to_dev(V[:2])).cpu().numpy()
    for r in range(2):
        check_rows(g[r], x, V[r], two_nu, "product", ell, 1.0, rows=rows, grad=True,
                   what=f"product nu={two_nu}/2 multilevel grad rhs {r}")


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
@pytest.mark.parametrize("n", [2, 64, 2049, 5000])
def test_product_d3_grad_all_rows(gpm, two_nu, n):
    """Lengthscale gradient of the d = 3 product form (product rule g1 k2 k3 + k1 g2 k3 +
    k1 k2 g3) by the separated sub-passes in two runs, every row, ties."""
    x = _pts(n, 3, 23 * n + two_nu, ties=(n % 2 == 1))
    v = np.random.default_rng(n + two_nu + 5).standard_normal(n)
    ell = (0.2, 0.3, 0.25)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 0.9, form=1))
    out = plan.kmvm_dlengthscale(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "product", ell, 0.9, grad=True,
               what=f"product d3 grad nu={two_nu}/2 n={n}")


def test_product_d3_grad_multilevel(gpm):
    """d = 3 product gradient with carried passes and outer levels > 10, 2 columns, rank-order
    entry bitwise equal to the user-order one."""
    n = 70_001
    x = _pts(n, 3, 99)
    V = np.random.default_rng(98).standard_normal((2, n))
    ell = (0.15, 0.25, 0.4)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, ell, 1.0, form=1))
    g = plan.kmvm_dlengthscale(to_dev(V)).cpu().numpy()
    rows = W.sample_rows(x, 128)
    for r in range(2):
        check_rows(g[r], x, V[r], 3, "product", ell, 1.0, rows=rows, grad=True,
                   what=f"product d3 multilevel grad rhs {r}")
    vr = plan.to_rank(to_dev(V[0]))
    gr = plan.from_rank(plan.kmvm_dlengthscale(vr, rank_order=True)).cpu().numpy()
    assert np.array_equal(gr, g[0])
    # deterministic: the two-run gradient repeats bitwise
    assert np.array_equal(plan.kmvm_dlengthscale(to_dev(V)).cpu().numpy(), g)


@pytest.mark.parametrize("two_nu", [5, 7, 9])
def test_high_nu_product_d2_kzx_and_gp(gpm, two_nu):
    """K_zx v on the union x U z (queries on top of data points included) and a CG + GLS
    solve with the d = 2 product kernel of order two_nu/2, against the oracle's dense rows
    and its dense-Cholesky GP (mean, alpha, beta)."""
    import oracle
    rng = np.random.default_rng(60 + two_nu)
    n, m = 2500, 600
    x = rng.random((n, 2))
    z = rng.random((m, 2))
    z[:40] = x[:40]
    ell = (0.15, 0.25)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.0, form=1))
    v = rng.standard_normal(n)
    out = plan.cross(to_dev(z)).kzx(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "product", ell, 1.0, z=z, what=f"kzx product nu={two_nu}/2")
    y = np.sin(4 * x[:, 0]) + x[:, 1] + 0.1 * rng.standard_normal(n)
    s2 = 0.05
    alpha, beta, info = plan.cg_solve(to_dev(y), s2, mean=gpm.MEAN_AFFINE, rtol=1e-10,
                                      max_iter=20000)
    ref = oracle.gp_dense(x, y, z, two_nu, "product", ell, 1.0, s2, mean="affine")
    assert info["relres_max"] <= 1e-10
    mu = plan.predict(to_dev(z), alpha, beta).cpu().numpy()
    # the solve against dense Cholesky (CG-tolerance bound, as test_cg_gls_predict_small_vs_dense)
    assert np.allclose(beta, ref["beta"], rtol=0, atol=1e-5)
    assert np.max(np.abs(mu - ref["mu"])) <= 1e-5 * max(1.0, np.max(np.abs(ref["mu"])))
    # the posterior mean given the GPU's alpha, beta: parity with the oracle's K_zx rows
    a = alpha.cpu().numpy()
    mu_or = oracle.kzx_rows(x, a, z, two_nu, "product", ell, 1.0) + \
        np.hstack([np.ones((m, 1)), z]) @ np.array(beta)
    assert np.max(np.abs(mu - mu_or)) <= 1e-9 * np.abs(a).max() * 50
