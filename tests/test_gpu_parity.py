"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): max|d| <= 1e-9 * ||K||_inf * ||v||_inf per MVM, with
||K||_inf the max absolute row sum over the checked rows; CG relative residual <= 1e-8.
Small cases check every row; full-size configs check seeded samples of rows
(workloads.sample_rows) in the launch configuration bench.py times.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from gpu_helpers import FORM, check_rows, to_dev

pytestmark = pytest.mark.gpu


def _points(kind, n, d, seed):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.random((n, d))
    if kind == "ties":           # coarse grid: many exact ties per coordinate + duplicates
        x = np.floor(rng.random((n, d)) * 17) / 17
        if n > 4:
            x[n // 2] = x[1]
        return x
    if kind == "normal":
        return rng.standard_normal((n, d))
    raise ValueError(kind)


D1_SIZES = [1, 2, 3, 7, 64, 1000, 4096, 7681, 20000]


@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("n", D1_SIZES)
@pytest.mark.parametrize("kind", ["uniform", "ties"])
def test_d1_all_rows(gpm, two_nu, n, kind):
    x = _points(kind, n, 1, n + two_nu)
    v = np.random.default_rng(n).standard_normal(n)
    ell = (0.07,)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.3))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "l1", ell, 1.3, what=f"d1 nu={two_nu}/2 n={n} {kind}")


@pytest.mark.parametrize("n", [1295, 1296, 1297, 2582, 2916, 4845, 2 * 27 * 4 * 7 + 1])
def test_d1_chunks_that_are_multiples_of_the_thread_items(gpm, n):
    """Chunks of 648 / 864 / 972 points are whole multiples of a thread's 27 items: no thread
    straddles the chunk end, and the first thread past it must still see the chunk's last
    point (a randomised sweep, tools/fuzz_parity.py, found its t_prev read from the shared
    tail window instead).  User and rank order, every row, and K_zx on a union."""
    rng = np.random.default_rng(n)
    x = rng.random((n, 1)); v = rng.standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1,), 1.0))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, 3, "l1", (0.1,), 1.0, what=f"d1 n={n} user order")
    outr = plan.from_rank(plan.kmvm_rank(plan.to_rank(to_dev(v)))).cpu().numpy()
    assert np.max(np.abs(outr - out)) <= 1e-13 * np.abs(out).max()
    z = rng.random((n // 3 + 1, 1))   # union sizes hit other chunk sizes
    cr = plan.cross(to_dev(z))
    check_rows(cr.kzx(to_dev(v)).cpu().numpy(), x, v, 3, "l1", (0.1,), 1.0, z=z, what=f"d1 n={n} kzx")
    cr.close()


@pytest.mark.parametrize("two_nu", [1, 5])
def test_d1_single_chunk_shapes(gpm, two_nu):
    """Every thread-block shape of the single-chunk kernel (512x15, 384x19, 256x27: the
    chunk splits at different thread / warp / part boundaries) against the oracle, equal
    to each other to rounding; option 0 = 2 (the removed multi-sub-tile path) is rejected."""
    n = 60000
    x = _points("normal", n, 1, 5)
    v = np.random.default_rng(6).standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, (0.02,)))
    rows = W.sample_rows(x, 1500)
    outs = []
    for shape in (0, 1, 2):
        plan.set_option(1, shape)
        assert plan.d1_path == 1 and plan.query(7) == shape
        out = plan.kmvm(to_dev(v)).cpu().numpy()
        check_rows(out, x, v, two_nu, "l1", (0.02,), 1.0, rows=rows, what=f"d1 shape {shape}")
        outs.append(out)
    for o in outs[1:]:
        assert np.max(np.abs(o - outs[0])) <= 1e-13 * np.abs(outs[0]).max()
    # user order, several columns per launch (the perm chunk shares the u buffer and is copied
    # again for every column's scatter): each column bitwise equal to its single-column apply
    V = np.random.default_rng(7).standard_normal((3, n))
    for shape in (0, 1, 2):
        plan.set_option(1, shape)
        multi = plan.kmvm(to_dev(V)).cpu().numpy()
        for c in range(3):
            assert np.array_equal(multi[c], plan.kmvm(to_dev(V[c])).cpu().numpy())
        check_rows(multi[2], x, V[2], two_nu, "l1", (0.02,), 1.0, rows=rows[:200],
                   what=f"d1 shape {shape} column 2 of 3")
    with pytest.raises(gpm.GPError) as e:
        plan.set_option(0, 2)
    assert e.value.name == "INVALID_ARG"


@pytest.mark.parametrize("n", [1, 7, 6912, 6913, 60001, 200_003])
@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
def test_d1_reduce_then_scan_path(gpm, n, two_nu):
    """The three-launch d = 1 path (sub-tile records, one-CTA carry scan, apply) forced at
    small sizes: user order against the oracle, rank order equal to user order to rounding
    (separately compiled kernels), multi-RHS columns bitwise equal to single columns."""
    import torch
    x = _points("normal" if n > 100 else "ties", n, 1, n + two_nu)
    V = np.random.default_rng(n).standard_normal((2, n))
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, (0.02,)))
    plan.set_option(0, 3)
    assert plan.d1_path == 3
    out = plan.kmvm(to_dev(V)).cpu().numpy()
    rows = W.sample_rows(x, 600) if n > 600 else None
    for c in range(2):
        check_rows(out[c], x, V[c], two_nu, "l1", (0.02,), 1.0, rows=rows,
                   what=f"d1 path 3 nu={two_nu}/2 n={n} col {c}")
    assert np.array_equal(plan.kmvm(to_dev(V[1])).cpu().numpy(), out[1])
    vr = plan.to_rank(to_dev(V[0]))
    o_r = plan.from_rank(plan.kmvm_rank(vr)).cpu().numpy()
    assert np.max(np.abs(o_r - out[0])) <= 1e-14 * max(np.abs(out[0]).max(), 1e-300)


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
def test_d1_reduce_then_scan_gradient(gpm, two_nu):
    n = 60001
    x = _points("normal", n, 1, 77)
    v = np.random.default_rng(78).standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, (0.02,)))
    plan.set_option(0, 3)
    out = plan.kmvm_dlengthscale(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "l1", (0.02,), 1.0, rows=W.sample_rows(x, 400), grad=True,
               what=f"d1 path 3 grad nu={two_nu}/2")


def test_config1_all_rows(gpm):
    c = W.CONFIGS[1]
    x = W.config_points(c)
    v = W.config_vector(c, 0)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(1, c.ell))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, 1, "l1", c.ell, 1.0, what="config1")


@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 1000, 2049, 5000])
def test_d2_all_rows(gpm, form, two_nu, n):
    x = _points("ties" if n % 2 else "uniform", n, 2, 10 * n + two_nu)
    v = np.random.default_rng(n + 1).standard_normal(n)
    ell = (0.1, 0.2)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 0.9, form=form))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, FORM[form], ell, 0.9, what=f"d2 {FORM[form]} nu={two_nu}/2 n={n}")


@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("n", [1, 2, 5, 64, 1000, 2049, 5000])
def test_d3_all_rows(gpm, two_nu, n):
    x = _points("ties" if n % 2 else "uniform", n, 3, 7 * n + two_nu)
    v = np.random.default_rng(n + 2).standard_normal(n)
    ell = (0.2, 0.3, 0.5)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.1))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "l1", ell, 1.1, what=f"d3 nu={two_nu}/2 n={n}")


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
@pytest.mark.parametrize("n", [1, 2, 5, 64, 1000, 2049, 5000])
def test_d3_product_all_rows(gpm, two_nu, n):
    """Product form at d = 3 (P:416 [eq product_kernel], P:487-509 [Prop 2]): the
    (p+1)^2 re-weighted passes per level against the dense definition, every row, ties."""
    x = _points("ties" if n % 2 else "uniform", n, 3, 9 * n + two_nu)
    v = np.random.default_rng(n + 4).standard_normal(n)
    ell = (0.2, 0.3, 0.5)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.1, form=1))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, two_nu, "product", ell, 1.1, what=f"d3 product nu={two_nu}/2 n={n}")


@pytest.mark.parametrize("two_nu,n,nrhs", [(3, 70_001, 2), (5, 33_000, 1), (3, 200_003, 1)])
def test_d3_product_multilevel_rows(gpm, two_nu, n, nrhs):
    """d = 3 product form with carried passes and outer levels > 10 (k_mid3, k_cp sub-passes),
    several right-hand sides, sampled rows; K_zx on a union plan."""
    rng = np.random.default_rng(n + two_nu)
    x = rng.random((n, 3))
    V = rng.standard_normal((nrhs, n))
    ell = (0.15, 0.25, 0.4)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 0.8, form=1))
    out = plan.kmvm(to_dev(V if nrhs > 1 else V[0])).cpu().numpy().reshape(nrhs, n)
    rows = W.sample_rows(x, 256)
    for c in range(nrhs):
        check_rows(out[c], x, V[c], two_nu, "product", ell, 0.8, rows=rows,
                   what=f"d3 product nu={two_nu}/2 n={n} col {c}")
    if n == 70_001:
        z = rng.random((500, 3))
        got = plan.predict(to_dev(z), to_dev(V[0])).cpu().numpy()
        check_rows(got, x, V[0], two_nu, "product", ell, 0.8, z=z, what="d3 product predict")


@pytest.mark.parametrize("d,form", [(1, 0), (2, 0), (2, 1), (3, 0), (3, 1)])
def test_kzx_all_rows(gpm, d, form):
    n, m = 3000, 700
    x = _points("uniform", n, d, 3 + d)
    z = _points("uniform", m, d, 4 + d)
    z[:50] = x[:50]                         # queries on top of data points
    v = np.random.default_rng(9).standard_normal(n)
    ell = (0.1, 0.2, 0.3)[:d]
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, ell, form=form))
    cr = plan.cross(to_dev(z))
    out = cr.kzx(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, 3, FORM[form], ell, 1.0, z=z, what=f"kzx d={d}")


def test_properties_linearity_symmetry_determinism(gpm):
    import torch
    n = 6000
    x = _points("uniform", n, 2, 1)
    ell = (0.1, 0.2)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, ell, form=1))
    rng = np.random.default_rng(2)
    u = to_dev(rng.standard_normal(n)); v = to_dev(rng.standard_normal(n))
    Ku, Kv = plan.kmvm(u), plan.kmvm(v)
    _, ab = oracle.kmvm_rows(x, np.ones(n), 3, "product", ell, rows=np.arange(0, n, 97), return_abs=True)
    Kn = ab.max()
    lhs = float(u @ Kv); rhs = float(v @ Ku)
    assert abs(lhs - rhs) <= 1e-9 * Kn * n * 5
    K2 = plan.kmvm(2 * u - 3 * v)
    assert float((K2 - (2 * Ku - 3 * Kv)).abs().max()) <= 1e-9 * Kn * 5 * 5
    # determinism: bitwise identical across repeated applies
    ref = plan.kmvm(u)
    for _ in range(20):
        assert torch.equal(plan.kmvm(u), ref)
    # multi-RHS equals separate applies
    V = torch.stack([u, v])
    KV = plan.kmvm(V)
    assert torch.equal(KV[0], Ku) and torch.equal(KV[1], Kv)


def test_d1_determinism_bitwise(gpm):
    import torch
    n = 300000
    x = _points("normal", n, 1, 3)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.05,)))
    v = to_dev(np.random.default_rng(1).standard_normal(n))
    ref = plan.kmvm(v)
    for _ in range(50):
        assert torch.equal(plan.kmvm(v), ref)


@pytest.mark.parametrize("d", [1, 2, 3])
def test_rank_order_operator(gpm, d):
    """gp_kmvm_rank on permuted vectors equals gp_kmvm; gp_permute round-trips bitwise."""
    import torch
    n = 9000 if d < 3 else 3000
    x = _points("uniform", n, d, 40 + d)
    v = to_dev(np.random.default_rng(d).standard_normal(n))
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.1, 0.2, 0.3)[:d]))
    vr = plan.to_rank(v)
    assert torch.equal(plan.from_rank(vr), v)
    out_r = plan.kmvm_rank(vr)
    assert torch.equal(plan.from_rank(out_r), plan.kmvm(v))


def test_host_buffers_e2e(gpm):
    n = 5000
    x = _points("uniform", n, 2, 8)
    v = np.random.default_rng(3).standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.1, 0.1)))
    out = np.empty(n)
    plan.kmvm_host(v, out)
    dev = plan.kmvm(to_dev(v)).cpu().numpy()
    assert np.array_equal(out, dev)


def test_errors(gpm):
    x = np.random.default_rng(0).random((100, 2))
    x[37, 1] = np.nan
    with pytest.raises(gpm.GPError) as e:
        gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.1)))
    assert e.value.name == "NONFINITE" and "row 37" in str(e.value)
    with pytest.raises(gpm.GPError) as e:
        gpm.Plan(to_dev(np.zeros((10, 3))), gpm.Kernel(4, (0.1,) * 3, form=1))
    assert e.value.name == "UNSUPPORTED"


# ------------------------------------------------------------------ solver (a9-a11)

def test_cg_gls_predict_small_vs_dense(gpm):
    c = W.scaled(W.CONFIGS[5], 2500, m=400)
    x = W.config_points(c); y = W.config_response(c, x); z = W.config_queries(c)
    s2 = c.noise_sigma ** 2
    ref = oracle.gp_dense(x, y, z, 3, "product", c.ell, 1.0, s2, mean="affine")
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, c.ell, form=1))
    alpha, beta, info = plan.cg_solve(to_dev(y), s2, mean=gpm.MEAN_AFFINE, rtol=1e-10)
    assert info["relres_max"] <= 1e-10
    alpha = alpha.cpu().numpy()
    # ||alpha - alpha*|| <= ||A^-1|| ||r|| <= ||r|| / sigma^2 (+ GLS propagation)
    assert np.allclose(beta, ref["beta"], rtol=0, atol=1e-6)
    assert np.max(np.abs(alpha - ref["alpha"])) <= 1e-10 * np.linalg.norm(y) / s2 * 10
    mu = plan.predict(to_dev(z), to_dev(alpha), beta).cpu().numpy()
    assert np.max(np.abs(mu - ref["mu"])) <= 1e-6
    # posterior mean from the GPU alpha/beta, checked against the oracle's K_zx rows
    mu_or = oracle.kzx_rows(x, alpha, z, 3, "product", c.ell, 1.0) + \
        np.hstack([np.ones((z.shape[0], 1)), z]) @ np.array(beta)
    assert np.max(np.abs(mu - mu_or)) <= 1e-9 * np.abs(alpha).max() * 50


@pytest.mark.parametrize("two_nu", [3, 5])
def test_cg_gls_predict_d3_product_vs_dense(gpm, two_nu):
    """Full GP inference on the d = 3 product form (PD, App B): CG + GLS with
    H = [1, x] + posterior mean against the dense oracle."""
    rng = np.random.default_rng(60 + two_nu)
    n, m = 2200, 300
    x = rng.random((n, 3)); z = rng.random((m, 3))
    y = 1 + 0.5 * x[:, 0] - 0.3 * x[:, 1] + 0.2 * x[:, 2] + np.sin(5 * x[:, 0]) * np.cos(3 * x[:, 2]) \
        + 0.1 * rng.standard_normal(n)
    ell = (0.2, 0.3, 0.25); s2 = 0.01
    ref = oracle.gp_dense(x, y, z, two_nu, "product", ell, 1.0, s2, mean="affine")
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, form=1))
    alpha, beta, info = plan.cg_solve(to_dev(y), s2, mean=gpm.MEAN_AFFINE, rtol=1e-10)
    assert info["relres_max"] <= 1e-10
    assert np.allclose(beta, ref["beta"], rtol=0, atol=1e-6)
    assert np.max(np.abs(alpha.cpu().numpy() - ref["alpha"])) <= 1e-10 * np.linalg.norm(y) / s2 * 10
    mu = plan.predict(to_dev(z), alpha, beta).cpu().numpy()
    assert np.max(np.abs(mu - ref["mu"])) <= 1e-6


@pytest.mark.parametrize("d", [1, 2])
def test_cg_solutions_and_ols_vs_dense(gpm, d, monkeypatch):
    """gp_cg_solve_ex by-products: the CG solutions X = [A^-1 y, A^-1 H] (user order) and
    beta_OLS against the dense oracle; the fused / graph-replayed iteration equals
    the unfused stream loop to rounding (GPM_CG_NOGRAPH runs the same kernels directly)."""
    c = W.scaled(W.CONFIGS[5], 1800, m=10)
    rng = np.random.default_rng(40 + d)
    x = rng.random((1800, d)); y = W.config_response(c, np.hstack([x, x])[:, :2])
    s2 = 0.01
    ell = (0.1,) * d
    ref = oracle.gp_dense(x, y, x[:3], 3, "product", ell, 1.0, s2, mean="affine")
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, ell, form=1))
    a, b, info = plan.cg_solve(to_dev(y), s2, rtol=1e-11, return_x=True, return_ols=True)
    X = info["X"].cpu().numpy()
    tol = 1e-11 * np.linalg.norm(y) / s2 * 100
    assert np.max(np.abs(X[0] - ref["A_inv_y"])) <= tol
    for j in range(1 + d):
        assert np.max(np.abs(X[1 + j] - ref["A_inv_H"][:, j])) <= tol * 10
    assert np.allclose(info["beta_ols"], ref["beta_ols"], rtol=1e-12, atol=1e-12)
    assert np.allclose(b, ref["beta"], rtol=0, atol=1e-7)
    monkeypatch.setenv("GPM_CG_NOGRAPH", "1")
    a2, b2, info2 = plan.cg_solve(to_dev(y), s2, rtol=1e-11)
    assert info2["iters"] == info["iters"]
    assert torch_equal_close(a, a2)


def torch_equal_close(a, b):
    import torch
    return bool(torch.equal(a, b))


def test_cg_no_mean_and_basis(gpm):
    rng = np.random.default_rng(4)
    x = rng.random((1500, 1)); y = np.sin(7 * x[:, 0]) + 0.1 * rng.standard_normal(1500)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.1,)))
    a0, b0, _ = plan.cg_solve(to_dev(y), 0.01, mean=gpm.MEAN_NONE, rtol=1e-10)
    ref = oracle.gp_dense(x, y, x[:5], 5, "l1", (0.1,), 1.0, 0.01, mean="none")
    assert b0 == [] and np.max(np.abs(a0.cpu().numpy() - ref["alpha"])) < 1e-6
    H = np.vstack([np.ones(1500), x[:, 0], x[:, 0] ** 2])
    a1, b1, _ = plan.cg_solve(to_dev(y), 0.01, mean=gpm.MEAN_BASIS, H=to_dev(H), rtol=1e-10)
    ref = oracle.gp_dense(x, y, x[:5], 5, "l1", (0.1,), 1.0, 0.01, mean="basis", H=H.T, Hz=H.T[:5])
    assert np.allclose(b1, ref["beta"], atol=1e-6)
    assert np.max(np.abs(a1.cpu().numpy() - ref["alpha"])) < 1e-6


def test_cg_breakdown_on_indefinite_l1(gpm):
    """L1 Matern-3/2 in d=2 is not PD (reading R4): CG must report BREAKDOWN."""
    x = W.uniform_points(2000, 2, 0); y = np.sin(3 * x[:, 0])
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.1), form=0))
    with pytest.raises(gpm.GPError) as e:
        plan.cg_solve(to_dev(y), 0.01, mean=gpm.MEAN_AFFINE, rtol=1e-8)
    assert e.value.name == "BREAKDOWN"


# ------------------------------------------------------------------ d >= 2 launch structure

@pytest.mark.parametrize("lb", ["0,0,0", "3,4,2", "5,7,6", "10,10,10"])
@pytest.mark.parametrize("d,two_nu,form", [(2, 3, 0), (2, 5, 1), (3, 5, 0), (3, 1, 0)])
def test_near_field_block_sizes(gpm, monkeypatch, lb, d, two_nu, form):
    """Every split of the D&C levels between exact near-field block sums, the fused
    scan kernels, the d=3 mid kernel and the carried multi-tile passes gives the same
    K.v (N = 6000 > 4 tiles: levels up to 13, l1 > 10 and l2 > 10 all exercised)."""
    monkeypatch.setenv("GPM_NEAR_LB", lb)
    n = 6000
    x = _points("ties", n, d, 300 + d)
    v = np.random.default_rng(5).standard_normal(n)
    ell = (0.1, 0.2, 0.3)[:d]
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, 1.0, form=form))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    rows = np.arange(0, n, 3)
    check_rows(out, x, v, two_nu, FORM[form], ell, 1.0, rows=rows, what=f"near lb={lb} d={d}")


@pytest.mark.parametrize("d", [1, 2, 3])
def test_multi_rhs_batches(gpm, d):
    """nrhs = 11 (> one batch of 8 columns) equals column-by-column applies bitwise."""
    import torch
    n = 3000
    x = _points("uniform", n, d, 70 + d)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.2, 0.3)[:d]))
    V = to_dev(np.random.default_rng(d).standard_normal((11, n)))
    KV = plan.kmvm(V)
    for c in (0, 7, 8, 10):
        assert torch.equal(KV[c], plan.kmvm(V[c].contiguous()))
    z = to_dev(_points("uniform", 500, d, 80 + d))
    cr = plan.cross(z)
    KZ = cr.kzx(V)
    for c in (0, 9):
        assert torch.equal(KZ[c], cr.kzx(V[c].contiguous()))
    ref = oracle.kzx_rows(x, V[9].cpu().numpy(), z.cpu().numpy(), 3, "l1", (0.1, 0.2, 0.3)[:d])
    assert np.max(np.abs(KZ[9].cpu().numpy() - ref)) < 1e-9 * np.abs(ref).max() * 50


@pytest.mark.parametrize("n", [3000, 3001, 200_003])
@pytest.mark.parametrize("nrhs", [2, 5])
def test_rank_order_multi_rhs_pipeline(gpm, n, nrhs):
    """d = 1 rank order with several columns in one launch: every column equals its
    single-column apply bitwise, over repeated launches (the exchange's record counts
    carry across launches); odd n exercises the non-bulk-copy loads."""
    import torch
    x = _points("normal", n, 1, 90 + nrhs)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.05,)))
    V = to_dev(np.random.default_rng(n + nrhs).standard_normal((nrhs, n)))
    VR = torch.stack([plan.to_rank(V[c].contiguous()) for c in range(nrhs)])
    for rep in range(3):   # repeated launches: the record counts carry across launches
        KR = plan.kmvm_rank(VR)
        for c in range(nrhs):
            assert torch.equal(KR[c], plan.kmvm_rank(VR[c].contiguous())), (rep, c)
    rows = workloads_rows(n)
    check_rows(plan.from_rank(KR[nrhs - 1]).cpu().numpy(), x, V[nrhs - 1].cpu().numpy(), 5, "l1",
               (0.05,), 1.0, rows=rows, what=f"pipeline n={n} nrhs={nrhs}")


def workloads_rows(n):
    return np.unique(np.concatenate([np.arange(0, min(n, 64)), np.arange(n - min(n, 64), n),
                                     np.random.default_rng(5).choice(n, min(n, 256), replace=False)]))


@pytest.mark.parametrize("d,ell", [(2, (0.6, 0.9)), (3, (0.7, 0.8, 0.9))])
def test_large_n_segments_over_256_tiles(gpm, d, ell):
    """N > 2^18: the top D&C node spans > 256 tiles (carry folds over many tile
    aggregates); long lengthscales make those far pairs matter."""
    n = 300_000
    x = _points("uniform", n, d, 900 + d)
    v = np.random.default_rng(11).standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, ell, 1.0))
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    rows = W.sample_rows(x, 256)
    check_rows(out, x, v, 3, "l1", ell, 1.0, rows=rows, what=f"large-n d={d}")


def test_host_buffers_pipelined_batch(gpm):
    """gp_kmvm_host with several pinned columns (pipelined copies) equals device applies."""
    import torch
    n = 30000
    x = _points("normal", n, 1, 12)
    V = torch.from_numpy(np.random.default_rng(4).standard_normal((7, n))).pin_memory()
    O = torch.empty_like(V).pin_memory()
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.05,)))
    plan.kmvm_host(V, O)
    dev = plan.kmvm(V.cuda()).cpu()
    assert torch.equal(O, dev)
    # pageable buffers take the plain path, same values
    O2 = np.empty((7, n))
    plan.kmvm_host(V.numpy().copy(), O2)
    assert np.array_equal(O2, dev.numpy())


def test_torch_allocator_hook(gpm):
    """gp_set_allocator through PyTorch's caching allocator: same results, memory from torch."""
    import torch
    x = _points("uniform", 20000, 2, 5)
    v = to_dev(np.random.default_rng(5).standard_normal(20000))
    ref = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.1))).kmvm(v)
    before = torch.cuda.memory_allocated()
    gpm.use_torch_allocator(True)
    try:
        plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.1)))
        out = plan.kmvm(v)
        assert torch.cuda.memory_allocated() > before + 20000 * 8
        assert torch.equal(out, ref)
        plan.close()
    finally:
        gpm.use_torch_allocator(False)


def test_predict_union_cache(gpm):
    """gp_predict caches the x U z structure (SURVEY §8(b) convention 4): a repeat call with
    the same z is bitwise equal to the first; z changed in place (same pointer, same m) is
    detected and gives the oracle's answer for the new points; a new m rebuilds."""
    import torch
    rng = np.random.default_rng(11)
    x = rng.random((3000, 2)); a = rng.standard_normal(3000)
    z = torch.from_numpy(rng.random((400, 2))).cuda()
    plan = gpm.Plan(to_dev(x), gpm.Kernel(3, (0.1, 0.2), form=1))
    ad = to_dev(a)
    m1 = plan.predict(z, ad, [0.5, 1.0, -1.0])
    m2 = plan.predict(z, ad, [0.5, 1.0, -1.0])
    assert torch.equal(m1, m2)
    z.mul_(0.5)   # in place: same pointer and m, new contents
    m3 = plan.predict(z, ad, None).cpu().numpy()
    zh = z.cpu().numpy()
    ref, ab = oracle.kzx_rows(x, a, zh, 3, "product", (0.1, 0.2), 1.0, return_abs=True)
    assert np.max(np.abs(m3 - ref)) <= 1e-9 * ab.max() * np.abs(a).max()
    m4 = plan.predict(z[:100].contiguous(), ad, None).cpu().numpy()
    assert np.max(np.abs(m4 - ref[:100])) <= 1e-9 * ab.max() * np.abs(a).max()
    plan.close()


@pytest.mark.parametrize("d,n,two_nu,form", [(2, 20000, 3, 0), (2, 9000, 3, 1), (3, 5000, 5, 0),
                                             (3, 70000, 3, 0), (3, 9000, 3, 1)])
@pytest.mark.parametrize("nshards", [2, 3, 5])
def test_sharded_apply_sums_to_kv(gpm, d, n, two_nu, form, nshards):
    """SURVEY §8(e) decomposition on one GPU: the shards of gp_kmvm_partial (tile and
    carried-pass item ranges of the D&C kernels) sum to the whole rank-order apply, for
    sizes with carried passes and (d = 3) outer levels above the tile; two columns."""
    import torch
    rng = np.random.default_rng(n + nshards)
    x = rng.random((n, d))
    ell = (0.2, 0.3, 0.4)[:d]
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell, form=form))
    V = torch.from_numpy(rng.standard_normal((2, n))).cuda()
    VR = torch.stack([plan.to_rank(V[i].contiguous()) for i in range(2)])
    full = plan.kmvm_rank(VR)
    acc = torch.zeros_like(full)
    for s in range(nshards):
        acc += plan.kmvm_partial(VR, s, nshards)
    assert torch.max(torch.abs(acc - full)).item() <= 1e-12 * torch.max(torch.abs(full)).item()
    assert torch.equal(plan.kmvm_rank(VR), full)   # back to the whole apply afterwards
    with pytest.raises(gpm.GPError):
        plan.kmvm_partial(VR, nshards, nshards)
    plan.close()
