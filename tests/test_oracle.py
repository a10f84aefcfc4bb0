"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Each pin is independent of the oracle's own formula (oracle/matern_oracle.c uses
the closed-form profiles of PAPER.md L1273-1275):
  * the Bessel-function definition of the Matern kernel (PAPER.md L1244-1253
    [eq matern_general, scaled_matern]) evaluated with mpmath at 50 digits;
  * the general half-integer coefficient formula (PAPER.md L1282 [eq matern_explicit])
    feeding exact geometric-series closed forms on equispaced grids;
  * the Kronecker identity of product kernels on tensor grids;
  * SPEC.md worked examples;
  * mpmath brute force at 40 digits on tiny inputs;
  * GLS special cases and invariants (symmetry, PD, subset rows).
"""
import math
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import oracle
import workloads as W


# ---------------------------------------------------------------- helpers (tests only)

def bessel_profile(two_nu, r, dps=50):
    """k_nu(r) from PAPER.md L1250 [eq matern_general] (modified Bessel K_nu), mpmath."""
    with mp.workdps(dps):
        nu = mp.mpf(two_nu) / 2
        r = mp.mpf(r)
        if r == 0:
            return mp.mpf(1)
        s = mp.sqrt(2 * nu) * r
        return s ** nu / (2 ** (nu - 1) * mp.gamma(nu)) * mp.besselk(nu, s)


def explicit_coeffs(p):
    """a_i of PAPER.md L1282 [eq matern_explicit] written for s = sqrt(2p+1)|u|:
    k(s) = sum_i a_i s^i e^{-s},  a_i = C(p,i) (2p-i)!/(2p)! 2^i (exact rationals)."""
    return [Fraction(math.comb(p, i) * math.factorial(2 * p - i) * 2 ** i, math.factorial(2 * p))
            for i in range(p + 1)]


def S_closed(q, n, rho):
    """sum_{k=0}^{n} k^q rho^k in closed form (q = 0, 1, 2)."""
    if q == 0:
        return (1 - rho ** (n + 1)) / (1 - rho)
    if q == 1:
        return rho * (1 - (n + 1) * rho ** n + n * rho ** (n + 1)) / (1 - rho) ** 2
    if q == 2:
        return rho * (1 + rho - (n + 1) ** 2 * rho ** n + (2 * n * n + 2 * n - 1) * rho ** (n + 1)
                      - n * n * rho ** (n + 2)) / (1 - rho) ** 3
    raise ValueError(q)


def equispaced_K1(n, delta, two_nu, ell):
    """(K 1)_j on x_i = i*delta, d = 1, from the closed forms (mpmath, 40 digits)."""
    p = (two_nu - 1) // 2
    a = explicit_coeffs(p)
    with mp.workdps(40):
        h = mp.sqrt(two_nu) * mp.mpf(delta) / mp.mpf(ell)
        rho = mp.e ** (-h)
        out = []
        for j in range(n):
            tot = mp.mpf(0)
            for q in range(p + 1):
                tot += mp.mpf(a[q].numerator) / a[q].denominator * h ** q * (
                    S_closed(q, j, rho) + S_closed(q, n - 1 - j, rho) - (1 if q == 0 else 0))
            out.append(tot)
        return np.array([float(t) for t in out])


# ---------------------------------------------------------------- pins

def test_closed_form_sums_exact():
    """S_q closed forms (used by the pins below) against exact rational sums."""
    rho = Fraction(3, 7)
    for q in range(3):
        for n in (0, 1, 2, 5, 9):
            direct = sum(Fraction(k) ** q * rho ** k for k in range(n + 1))
            assert S_closed(q, n, rho) == direct


def test_explicit_coeffs_match_paper_table():
    """eq matern_explicit (L1282) reproduces the displayed k_{1/2..9/2} (L1273-1277)."""
    assert explicit_coeffs(0) == [1]
    assert explicit_coeffs(1) == [1, 1]
    assert explicit_coeffs(2) == [1, 1, Fraction(1, 3)]
    # k_{7/2}: 1 + sqrt7 u + 14/5 u^2 + 7 sqrt7/15 u^3 -> in s = sqrt7 u: 1, 1, 2/5, 1/15
    assert explicit_coeffs(3) == [1, 1, Fraction(2, 5), Fraction(1, 15)]
    # k_{9/2}: 1 + 3u + 27/7 u^2 + 18/7 u^3 + 27/35 u^4 -> in s = 3u: 1, 1, 3/7, 2/21, 1/105
    assert explicit_coeffs(4) == [1, 1, Fraction(3, 7), Fraction(2, 21), Fraction(1, 105)]


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
def test_profile_against_bessel_definition(two_nu):
    for r in [0.0, 1e-3, 0.05, 0.3, 1.0, 2.5, 7.0, 30.0]:
        ref = float(bessel_profile(two_nu, r))
        got = oracle.kernel_value(two_nu, "l1", [1.0], 1.0, [0.0], [r])
        # exp(-s) amplifies the rounding of s = sqrt(2nu) r: relative error ~ s * eps
        rel = 4.5e-16 * (4.0 + math.sqrt(two_nu) * r)
        assert got == pytest.approx(ref, rel=rel, abs=1e-300), (two_nu, r)


def test_spec_worked_examples():
    # k_{1/2}(1) = 0.36787944117; k(0) = s^2; L1 d=2 u=(1,1) -> e^-2
    assert oracle.kernel_value(1, "l1", [1.0], 1.0, [0.0], [1.0]) == pytest.approx(0.36787944117, abs=1e-11)
    assert oracle.kernel_value(5, "l1", [0.7], 1.9, [0.3], [0.3]) == pytest.approx(1.9 ** 2, rel=1e-15)
    assert oracle.kernel_value(1, "l1", [1.0, 1.0], 1.0, [0, 0], [1, 1]) == pytest.approx(0.13533528, abs=1e-8)
    # x=(0,1), y=(1,1), nu=1/2, s=l=1 -> (1+e^-1, 1+e^-1)
    out = oracle.kmvm_rows(np.array([0.0, 1.0]), np.ones(2), 1, "l1", [1.0], 1.0)
    assert np.allclose(out, 1 + math.exp(-1), rtol=1e-15)
    # N=1 -> s^2 v_1
    assert oracle.kmvm_rows(np.array([0.4]), np.array([2.5]), 3, "l1", [0.1], 2.0)[0] == pytest.approx(10.0)


@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("n,delta,ell", [(37, 0.05, 0.3), (200, 0.011, 0.05), (64, 0.4, 0.2)])
def test_equispaced_geometric_series(two_nu, n, delta, ell):
    """d = 1, equispaced x, v = 1: the geometric-series closed form named in north_star."""
    x = np.arange(n) * delta
    got = oracle.kmvm_rows(x, np.ones(n), two_nu, "l1", [ell], 1.0)
    ref = equispaced_K1(n, delta, two_nu, ell)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("two_nu", [1, 3, 5])
def test_kzx_offset_queries_closed_form(two_nu):
    """K_zx 1 with queries halfway between equispaced data points (closed form)."""
    n, delta, ell = 50, 0.03, 0.15
    p = (two_nu - 1) // 2
    a = explicit_coeffs(p)
    x = np.arange(n) * delta
    z = (np.arange(n - 1) + 0.5) * delta
    got = oracle.kzx_rows(x, np.ones(n), z, two_nu, "l1", [ell], 1.0)
    with mp.workdps(40):
        h = mp.sqrt(two_nu) * mp.mpf(delta) / ell
        rho = mp.e ** (-h)
        ref = []
        for j in range(n - 1):
            tot = mp.mpf(0)
            for q in range(p + 1):
                for m in range(q + 1):
                    c = mp.mpf(a[q].numerator) / a[q].denominator * math.comb(q, m) * mp.mpf(0.5) ** (q - m)
                    tot += c * h ** q * (S_closed(m, j, rho) + S_closed(m, n - 2 - j, rho))
            ref.append(float(mp.sqrt(rho) * tot))
    ref = np.array(ref)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(ref)


@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("d", [2, 3])
def test_product_kronecker_tensor_grid(two_nu, d):
    """Product kernel on a tensor grid, v = 1: K 1 = (x)_k (K_k 1)  (Kronecker identity)."""
    ns = [9, 7, 5][:d]
    deltas = [0.05, 0.13, 0.02][:d]
    ells = [0.1, 0.35, 0.07][:d]
    axes = [np.arange(nk) * dk for nk, dk in zip(ns, deltas)]
    grid = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, d)
    got = oracle.kmvm_rows(grid, np.ones(grid.shape[0]), two_nu, "product", ells, 1.3)
    fac = [equispaced_K1(nk, dk, two_nu, lk) for nk, dk, lk in zip(ns, deltas, ells)]
    ref = 1.3 ** 2 * np.einsum("i,j->ij", fac[0], fac[1]).ravel() if d == 2 else \
        1.3 ** 2 * np.einsum("i,j,k->ijk", fac[0], fac[1], fac[2]).ravel()
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(ref)
    if two_nu == 1:   # nu = 1/2: L1 and product coincide
        got_l1 = oracle.kmvm_rows(grid, np.ones(grid.shape[0]), 1, "l1", ells, 1.3)
        assert np.max(np.abs(got_l1 - ref)) <= 1e-13 * np.max(ref)


@pytest.mark.parametrize("form", ["l1", "product"])
@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_bruteforce_mpmath(form, two_nu, d):
    """Tiny N: oracle vs a 40-digit dense sum built on the Bessel definition."""
    rng = np.random.default_rng(100 * d + two_nu)
    n = 9
    x = rng.random((n, d))
    x[3] = x[1]                       # an exact duplicate
    x[5, 0] = x[2, 0]                 # a partial tie
    v = rng.standard_normal(n)
    ell = [0.3, 0.5, 0.2][:d]
    sig = 0.8
    got, ab = oracle.kmvm_rows(x, v, two_nu, form, ell, sig, return_abs=True)
    with mp.workdps(40):
        ref = []
        for j in range(n):
            tot = mp.mpf(0)
            for i in range(n):
                if form == "l1":
                    r = sum(abs(mp.mpf(x[i, k]) - mp.mpf(x[j, k])) / mp.mpf(ell[k]) for k in range(d))
                    kv = bessel_profile(two_nu, r, 40)
                else:
                    kv = mp.mpf(1)
                    for k in range(d):
                        kv *= bessel_profile(two_nu, abs(mp.mpf(x[i, k]) - mp.mpf(x[j, k])) / mp.mpf(ell[k]), 40)
                tot += mp.mpf(v[i]) * mp.mpf(sig) ** 2 * kv
            ref.append(float(tot))
    tol = 1e-14 * np.max(ab) * np.max(np.abs(v))
    assert np.max(np.abs(got - np.array(ref))) <= tol


def test_unit_vector_gives_column():
    """v = e_j returns column j of K, entry by entry."""
    rng = np.random.default_rng(4)
    x = rng.random((40, 2)); ell = [0.2, 0.4]
    j = 17
    e = np.zeros(40); e[j] = 1.0
    col = oracle.kmvm_rows(x, e, 5, "l1", ell, 1.0)
    for i in range(40):
        assert col[i] == oracle.kernel_value(5, "l1", ell, 1.0, x[i], x[j])


@pytest.mark.parametrize("form", ["l1", "product"])
def test_symmetry_linearity_rows(form):
    rng = np.random.default_rng(7)
    x = rng.random((300, 2)); ell = [0.1, 0.2]
    u = rng.standard_normal(300); v = rng.standard_normal(300)
    Ku, ab = oracle.kmvm_rows(x, u, 3, form, ell, return_abs=True)
    Kv = oracle.kmvm_rows(x, v, 3, form, ell)
    Knorm = ab.max()
    assert abs(u @ Kv - v @ Ku) <= 1e-12 * Knorm * (np.abs(u).sum() * np.abs(v).max() + np.abs(v).sum() * np.abs(u).max())
    K2 = oracle.kmvm_rows(x, 2.0 * u - 3.0 * v, 3, form, ell)
    assert np.max(np.abs(K2 - (2 * Ku - 3 * Kv))) <= 1e-12 * Knorm * 5 * max(np.abs(u).max(), np.abs(v).max())
    rows = np.array([0, 5, 299, 17])
    assert np.array_equal(oracle.kmvm_rows(x, u, 3, form, ell, rows=rows), Ku[rows])
    # K_zx with z = a subset of x equals those rows of K v
    assert np.array_equal(oracle.kzx_rows(x, u, x[rows], 3, form, ell), Ku[rows])


def test_anisotropic_scaling_invariance():
    """Scaling coordinate k and l_k by the same factor leaves K unchanged (reading R2)."""
    rng = np.random.default_rng(9)
    x = rng.random((100, 3)); v = rng.standard_normal(100)
    ell = np.array([0.2, 0.3, 0.5]); c = np.array([3.0, 0.25, 1.0])
    for form in ("l1", "product"):
        a = oracle.kmvm_rows(x, v, 5, form, ell)
        b = oracle.kmvm_rows(x * c, v, 5, form, ell * c)
        assert np.max(np.abs(a - b)) <= 1e-12 * np.abs(a).max()


def test_positive_definiteness_readings():
    """PD for product forms and nu=1/2 (App B); L1 nu>=3/2, d=2 is indefinite
    (reading R4) -- asserted so the reading stays documented."""
    x = W.uniform_points(600, 2, 0)
    for two_nu, form in [(1, "l1"), (3, "product"), (5, "product")]:
        K = oracle.dense_kernel(x, x, two_nu, form, [0.1, 0.1])
        w = np.linalg.eigvalsh(K)
        assert w[0] > -1e-10 * w[-1], (two_nu, form, w[0])
    K = oracle.dense_kernel(x, x, 3, "l1", [0.1, 0.1])
    assert np.linalg.eigvalsh(K)[0] < -1e-3


def test_gls_special_cases():
    rng = np.random.default_rng(11)
    x = rng.random((150, 2)); z = rng.random((20, 2))
    beta_star = np.array([1.0, 0.5, -0.3])
    H = np.hstack([np.ones((150, 1)), x])
    # y = H beta* exactly -> GLS returns beta* (S:440); alpha = 0 -> mu = h(z)^T beta*
    r = oracle.gp_dense(x, H @ beta_star, z, 3, "product", [0.1, 0.1], 1.0, 0.01)
    assert np.allclose(r["beta"], beta_star, rtol=0, atol=1e-10)
    assert np.max(np.abs(r["alpha"])) < 1e-9
    # outputscale -> 0: GLS -> OLS
    y = H @ beta_star + 0.1 * rng.standard_normal(150)
    r = oracle.gp_dense(x, y, z, 3, "product", [0.1, 0.1], 1e-7, 0.01)
    assert np.allclose(r["beta"], r["beta_ols"], atol=1e-10)
    # OLS recovers noiseless affine coefficients
    assert np.allclose(oracle.ols(H, H @ beta_star), beta_star, atol=1e-12)
    # basis mean with H = [1, x] equals the affine mean
    r1 = oracle.gp_dense(x, y, z, 3, "product", [0.1, 0.1], 1.0, 0.01, mean="affine")
    r2 = oracle.gp_dense(x, y, z, 3, "product", [0.1, 0.1], 1.0, 0.01, mean="basis",
                         H=H, Hz=np.hstack([np.ones((20, 1)), z]))
    assert np.allclose(r1["mu"], r2["mu"], atol=1e-12)


def test_gp_solution_and_interpolation():
    rng = np.random.default_rng(12)
    x = rng.random((200, 2)); y = np.sin(4 * x[:, 0]) + x[:, 1]
    # (K + s^2 I) alpha = y - H beta, checked with the row oracle (not the dense matrix)
    r = oracle.gp_dense(x, y, x[:5], 3, "product", [0.2, 0.2], 1.0, 0.04)
    H = np.hstack([np.ones((200, 1)), x])
    Ka = oracle.kmvm_rows(x, r["alpha"], 3, "product", [0.2, 0.2])
    assert np.max(np.abs(Ka + 0.04 * r["alpha"] - (y - H @ r["beta"]))) < 1e-9
    # near-interpolation at the data as sigma -> 0
    r = oracle.gp_dense(x, y, x[:10], 3, "product", [0.2, 0.2], 1.0, 1e-9)
    assert np.max(np.abs(r["mu"] - y[:10])) < 1e-5
    # far field: K_zx -> 0 and mu(z) -> h(z)^T beta
    zf = np.array([[1e4, 1e4]])
    r = oracle.gp_dense(x, y, zf, 3, "product", [0.2, 0.2], 1.0, 0.04)
    assert r["mu"][0] == pytest.approx(r["beta"] @ np.array([1.0, 1e4, 1e4]), rel=1e-12)


def test_workloads_recipes():
    c3 = W.scaled(W.CONFIGS[3], 5000, m=100)
    x = W.config_points(c3)
    assert x.shape == (5000, 2)
    u, counts = np.unique(x, axis=0, return_counts=True)
    assert 5000 - u.shape[0] == 50          # 1% exact duplicates
    assert np.array_equal(x, W.config_points(c3))
    x4 = W.config_points(W.scaled(W.CONFIGS[4], 2000))
    assert x4.shape == (2000, 3)
    rows = W.sample_rows(x4, 256)
    assert rows.size == 256 and np.all(np.diff(rows) > 0)
    assert int(np.argmax(x4[:, 2])) in set(rows.tolist())


# ---------------------------------------------------------------- lengthscale gradient (f2)

def explicit_dcoeffs(p):
    """Coefficients c_i of u^i in -k'_{p+1/2}(u) e^{sqrt(2p+1) u}
    [eq dmatern_explicit_dl], returned as c_i / (2p+1)^{i/2} in s = sqrt(2p+1) u units
    (exact rationals; the sqrt(2p+1) factors cancel to (2p+1)^{(i+1)/2 - i/2} = sqrt(2p+1)
    overall, which is dropped: -k'(u) = sqrt(2p+1) sum_i c_i s^i e^{-s})."""
    return [Fraction(0)] + [Fraction(i * math.comb(p, i) * math.factorial(2 * p - i) * 2 ** i,
                                     (2 * p - i) * math.factorial(2 * p))
                            for i in range(1, p + 1)]


def test_dmatern_explicit_matches_paper_table_and_derivative():
    """eq dmatern_explicit_dl (L1327) reproduces the displayed k'_{3/2..9/2} (L1321-1324)
    and equals the exact derivative of eq matern_explicit (L1282).  For p = 0 the general
    formula is an empty sum while eq dmatern12_dl (L1320) prints -e^{-u}: DESIGN.md reading
    R11 takes the displayed formula."""
    # -k'(s) in s units from differentiating sum_i a_i s^i e^{-s}: sum_i (a_i - (i+1) a_{i+1}) s^i
    for p in range(1, 5):
        a = explicit_coeffs(p) + [Fraction(0)]
        deriv = [a[i] - (i + 1) * a[i + 1] for i in range(p + 1)]
        assert explicit_dcoeffs(p) == deriv, p
    # displayed table, e.g. k'_{5/2}(u) = -(5/3 u + 5 sqrt5/3 u^2) e^{-sqrt5 u}:
    # in s = sqrt5 u: -k' = sqrt5 (1/3 s + 1/3 s^2) e^{-s}
    assert explicit_dcoeffs(1) == [0, 1]
    assert explicit_dcoeffs(2) == [0, Fraction(1, 3), Fraction(1, 3)]
    # k'_{7/2}: 7/5 u + 7 sqrt7/5 u^2 + 49/15 u^3 -> /sqrt7 in s: 1/5 s, 1/5 s^2, 1/15 s^3
    assert explicit_dcoeffs(3) == [0, Fraction(1, 5), Fraction(1, 5), Fraction(1, 15)]
    assert explicit_dcoeffs(0) == [0]


def bessel_dprofile_scaled(two_nu, r, dps=50):
    """-r k_nu'(r) from the Bessel definition: mpmath high-precision numerical derivative."""
    with mp.workdps(dps):
        r = mp.mpf(r)
        if r == 0:
            return mp.mpf(0)
        # the profile must run at a higher precision than diff's own (it raises it)
        return -r * mp.diff(lambda t: bessel_profile(two_nu, t, 3 * dps), r)


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
def test_dprofile_against_bessel_derivative(two_nu):
    for r in [0.0, 1e-3, 0.05, 0.3, 1.0, 2.5, 7.0, 30.0]:
        ref = float(bessel_dprofile_scaled(two_nu, r))
        got = oracle.dkernel_value(two_nu, "l1", [1.0], 1.0, [0.0], [r])
        rel = 4.5e-16 * (6.0 + 2 * math.sqrt(two_nu) * r)
        assert got == pytest.approx(ref, rel=rel, abs=1e-300), (two_nu, r)


@pytest.mark.parametrize("two_nu", [1, 3, 5, 7, 9])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_dkmvm_bruteforce_lengthscale_derivative(two_nu, d):
    """Tiny N: l dK/dl v (every l_k scaled together) vs the 40-digit derivative
    d/dc [sum_i v_i s^2 k_nu(sum_k |dx_k| / (c l_k))] at c = 1 on the Bessel definition."""
    rng = np.random.default_rng(300 + 10 * d + two_nu)
    n = 8
    x = rng.random((n, d))
    x[3] = x[1]
    v = rng.standard_normal(n)
    ell = [0.3, 0.5, 0.2][:d]
    sig = 1.3
    got, ab = oracle.dkmvm_rows(x, v, two_nu, "l1", ell, sig, return_abs=True)
    with mp.workdps(40):
        ref = []
        for j in range(n):
            def f(c):
                tot = mp.mpf(0)
                for i in range(n):
                    r = sum(abs(mp.mpf(x[i, k]) - mp.mpf(x[j, k])) / (c * mp.mpf(ell[k]))
                            for k in range(d))
                    tot += mp.mpf(v[i]) * mp.mpf(sig) ** 2 * bessel_profile(two_nu, r, 120)
                return tot
            ref.append(float(mp.diff(f, mp.mpf(1))))
    tol = 1e-14 * np.max(ab) * np.max(np.abs(v))
    assert np.max(np.abs(got - np.array(ref))) <= tol
    # zero on the diagonal: duplicates and the self pair contribute nothing
    e = np.zeros(n); e[1] = 1.0
    col = oracle.dkmvm_rows(x, e, two_nu, "l1", ell, sig)
    assert col[1] == 0.0 and col[3] == 0.0


@pytest.mark.parametrize("two_nu", [1, 3, 5])
@pytest.mark.parametrize("d", [2, 3])
def test_dkmvm_product_form_lengthscale_derivative(two_nu, d):
    """Product form: 40-digit d/dc of prod_k k(|dx_k| / (c l_k)) on the Bessel definition."""
    rng = np.random.default_rng(400 + 10 * d + two_nu)
    n = 7
    x = rng.random((n, d))
    v = rng.standard_normal(n)
    ell = [0.3, 0.5, 0.2][:d]
    got, ab = oracle.dkmvm_rows(x, v, two_nu, "product", ell, 0.9, return_abs=True)
    with mp.workdps(40):
        ref = []
        for j in range(n):
            def f(c):
                tot = mp.mpf(0)
                for i in range(n):
                    kv = mp.mpf(1)
                    for k in range(d):
                        kv *= bessel_profile(two_nu, abs(mp.mpf(x[i, k]) - mp.mpf(x[j, k])) /
                                             (c * mp.mpf(ell[k])), 120)
                    tot += mp.mpf(v[i]) * mp.mpf(0.9) ** 2 * kv
                return tot
            ref.append(float(mp.diff(f, mp.mpf(1))))
    assert np.max(np.abs(got - np.array(ref))) <= 1e-14 * np.max(ab) * np.max(np.abs(v))
