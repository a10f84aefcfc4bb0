"""Large sizes (the 'maximum sizes' edge cases): d = 1 beyond the single-launch limit
(multi-sub-tile path), d = 2 / d = 3 at several million points -- sampled rows against the
oracle, in the launch configuration of the public API."""
import numpy as np
import pytest

import workloads as W
from gpu_helpers import check_rows, to_dev

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,n,two_nu", [(1, 8_000_000, 3), (1, 3_000_000, 5), (2, 4_000_000, 3),
                                        (3, 2_000_000, 5)])
def test_large_n_sampled_rows(gpm, d, n, two_nu):
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d)) if d == 1 else rng.random((n, d))
    v = rng.standard_normal(n)
    ell = (0.05, 0.05, 0.1)[:d] if d > 1 else (0.01,)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(two_nu, ell))
    if d == 1:
        assert plan.d1_path == 3                   # beyond 148 x 7936 points: reduce-then-scan
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    rows = W.sample_rows(x, 96)
    check_rows(out, x, v, two_nu, "l1", ell, 1.0, rows=rows, what=f"large d={d} n={n}")
    plan.close()


def test_d1_two_pow_20_single_chunk(gpm):
    """N = 2^20 is above the default shape's capacity (#SMs x 6912): the automatic choice
    takes the 256 x 30 shape (#SMs x 7680) and keeps the single-launch kernel."""
    n = 1 << 20
    rng = np.random.default_rng(20)
    x = rng.random((n, 1)); v = rng.standard_normal(n)
    plan = gpm.Plan(to_dev(x), gpm.Kernel(5, (0.1,)))
    assert plan.d1_path == 1 and plan.query(7) == 1
    out = plan.kmvm(to_dev(v)).cpu().numpy()
    check_rows(out, x, v, 5, "l1", (0.1,), 1.0, rows=W.sample_rows(x, 256), what="d1 2^20")
    vr = plan.to_rank(to_dev(v))
    o2 = plan.from_rank(plan.kmvm_rank(vr)).cpu().numpy()
    assert np.max(np.abs(o2 - out)) <= 1e-13 * np.abs(out).max()
    plan.close()
