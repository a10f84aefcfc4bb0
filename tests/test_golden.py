"""Golden fixtures (tests/golden/, each line cited to PAPER.md or SPEC.md) against the
CPU oracle (CPU tests) and against the CUDA path through the C ABI (gpu tests).

The profile tables are the paper's printed closed forms (eq matern_1_2 .. matern_9_2,
eq dmatern12_dl .. dmatern92_dl), not the general formula the oracle is built from, so
they pin the oracle's coefficients independently of its own code.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
U_GRID = [0.0, 1e-3, 0.1, 0.5, 1.0, 2.0, 5.0, 20.0]


def _expr(s):
    """Value of an exact expression made of rationals, '*' and sqrt(k) (fixture syntax)."""
    val = 1.0
    for f in s.strip().split("*"):
        f = f.strip()
        if f.startswith("sqrt(") and "/" in f:                    # sqrt(k)/m
            root, den = f.split("/")
            val *= math.sqrt(int(root[5:-1])) / int(den)
        elif f.startswith("sqrt("):
            val *= math.sqrt(int(f[5:-1]))
        else:
            val *= float(Fraction(f))
    return val


def _table(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        if line.strip() and not line.startswith("#"):
            two_nu, rate, coefs = (c.strip() for c in line.split("|"))
            rows.append((int(two_nu), _expr(rate), [_expr(c) for c in coefs.split(";")]))
    return rows


def _profile(rate, c, u):
    return sum(ci * u ** i for i, ci in enumerate(c)) * math.exp(-rate * u)


@pytest.mark.parametrize("row", _table("paper_matern_profiles.txt"), ids=lambda r: f"2nu={r[0]}")
def test_oracle_profile_matches_paper_table(row):
    two_nu, rate, c = row
    for u in U_GRID:
        want = _profile(rate, c, u)
        got = oracle.kernel_value(two_nu, "l1", [1.0], 1.0, [0.0], [u])
        assert got == pytest.approx(want, rel=1e-14, abs=1e-300), (two_nu, u)


@pytest.mark.parametrize("row", _table("paper_matern_derivatives.txt"), ids=lambda r: f"2nu={r[0]}")
def test_oracle_lengthscale_derivative_matches_paper_table(row):
    # R11: l dK/dl = -s^2 u k'(u) (eq dkernel_dl times l), u = |x - y| / l
    two_nu, rate, d = row
    for u in U_GRID:
        kprime = -_profile(rate, d, u)
        got = oracle.dkernel_value(two_nu, "l1", [1.0], 1.0, [0.0], [u])
        assert got == pytest.approx(-u * kprime, rel=1e-13, abs=1e-300), (two_nu, u)


def _examples():
    out = []
    for line in open(os.path.join(GOLD, "spec_worked_examples.txt")):
        if line.strip() and not line.startswith("#"):
            out.append([c.strip() for c in line.split("|")])
    return out


def _floats(s):
    return [float(v) for v in s.split(",")]


@pytest.mark.parametrize("ex", _examples(), ids=lambda e: "-".join(e[:3]))
def test_oracle_spec_worked_examples(ex):
    if ex[0] == "kernel":
        _, two_nu, form, s, ell, u, val, tol = ex
        u = _floats(u)
        got = oracle.kernel_value(int(two_nu), form, _floats(ell), float(s), [0.0] * len(u), u)
        assert abs(got - float(val)) <= float(tol)
    else:
        _, two_nu, form, s, ell, xs, y, want, tol = ex
        x = np.array([_floats(p) for p in xs.split(";")])
        got = oracle.kmvm_rows(x, np.array(_floats(y)), int(two_nu), form, _floats(ell), float(s))
        assert np.max(np.abs(got - np.array(_floats(want)))) <= float(tol)


@pytest.mark.gpu
@pytest.mark.parametrize("row", _table("paper_matern_profiles.txt"), ids=lambda r: f"2nu={r[0]}")
def test_gpu_profile_matches_paper_table(gpm, row):
    """Column 0 of K on points {0} u U_GRID (v = e_0) is the printed profile (d = 1)."""
    import torch
    two_nu, rate, c = row
    x = np.array([0.0] + U_GRID[1:])[:, None]
    v = np.zeros(x.shape[0]); v[0] = 1.0
    plan = gpm.Plan(torch.from_numpy(x).cuda(), gpm.Kernel(two_nu, (1.0,), 1.0))
    out = plan.kmvm(torch.from_numpy(v).cuda()).cpu().numpy()
    plan.close()
    want = np.array([_profile(rate, c, u) for u in x[:, 0]])
    assert np.max(np.abs(out - want)) <= 1e-14


@pytest.mark.gpu
@pytest.mark.parametrize("ex", [e for e in _examples() if e[0] == "mvm"], ids=lambda e: "-".join(e[:3]))
def test_gpu_spec_worked_examples(gpm, ex):
    import torch
    _, two_nu, form, s, ell, xs, y, want, tol = ex
    x = np.array([_floats(p) for p in xs.split(";")])
    plan = gpm.Plan(torch.from_numpy(x).cuda(),
                    gpm.Kernel(int(two_nu), tuple(_floats(ell)), float(s),
                               form=gpm.FORM_PRODUCT if form == "product" else 0))
    got = plan.kmvm(torch.from_numpy(np.array(_floats(y))).cuda()).cpu().numpy()
    plan.close()
    assert np.max(np.abs(got - np.array(_floats(want)))) <= float(tol)
