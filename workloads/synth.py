"""Seeded input generators for the five BASELINE.json configs (and scaled-down copies).

Recipe:
  * geometry and targets of config c come from ``numpy.random.default_rng(c-1)``;
  * the vector of apply r comes from ``default_rng([c-1, 1000+r]).standard_normal(N)``;
  * every array is float64, C-contiguous, points row-major (N x d).

The paper's own workloads are synthetic too (x ~ U[0,1]^d, N = 2e4..2e5,
PAPER.md L721-724 [§3.1]); its one real dataset (L784-786) is not used.
Nothing here evaluates a kernel or solves anything.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Config", "CONFIGS", "config_points", "config_vector", "config_queries",
    "config_response", "sample_rows", "uniform_points", "scaled",
]


@dataclass(frozen=True)
class Config:
    idx: int                    # 1..5, BASELINE.json configs[idx-1]
    name: str
    d: int
    n: int
    two_nu: tuple               # 2*nu values exercised (1, 3, 5)
    form: str                   # "l1" or "product"
    ell: tuple                  # per-dimension lengthscale
    m: int = 0                  # number of query points (K_zx / predict)
    applies: int = 1            # repeated applies with fresh v
    noise_sigma: float = 0.0    # sigma of the nugget (config 5)
    extra_forms: tuple = field(default_factory=tuple)


CONFIGS = {
    1: Config(1, "d1_n4096_nu12", 1, 4096, (1,), "l1", (0.3,), applies=1),
    2: Config(2, "d1_n1e6_nu32_nu52", 1, 1_000_000, (3, 5), "l1", (0.05,), applies=100),
    3: Config(3, "d2_n2e5_nu32_ties_kzx", 2, 200_000, (3,), "l1", (0.1, 0.2), m=20_000,
              extra_forms=("product",)),
    4: Config(4, "d3_n5e5_nu52_gmm", 3, 500_000, (5,), "l1", (0.2, 0.3, 0.5), applies=50),
    5: Config(5, "d2_n3e5_gp_nu32_product", 2, 300_000, (3,), "product", (0.1, 0.1),
              m=10_000, noise_sigma=0.1),
}


def scaled(cfg: Config, n: int, m: int | None = None) -> Config:
    """Same recipe as ``cfg`` at a smaller N (for oracle-sized parity cases)."""
    return Config(cfg.idx, cfg.name + f"_n{n}", cfg.d, n, cfg.two_nu, cfg.form, cfg.ell,
                  m=cfg.m if m is None else m, applies=cfg.applies,
                  noise_sigma=cfg.noise_sigma, extra_forms=cfg.extra_forms)


def uniform_points(n: int, d: int, seed) -> np.ndarray:
    return np.ascontiguousarray(np.random.default_rng(seed).random((n, d)))


def config_points(cfg: Config) -> np.ndarray:
    """Data points x (N x d) of a config, following BASELINE.json configs[idx-1]."""
    rng = np.random.default_rng(cfg.idx - 1)
    n, d = cfg.n, cfg.d
    if cfg.idx == 1:
        x = rng.random((n, 1))
    elif cfg.idx == 2:
        x = rng.standard_normal((n, 1))
    elif cfg.idx == 3:
        # 1% exact duplicates (ties), shuffled in
        n_dup = max(n // 100, 1) if n >= 2 else 0
        base = rng.random((n - n_dup, 2))
        dup = rng.choice(n - n_dup, n_dup, replace=False) if n_dup else np.zeros(0, int)
        x = rng.permutation(np.vstack([base, base[dup]]))
    elif cfg.idx == 4:
        means = rng.random((16, 3))
        comp = rng.integers(0, 16, n)
        x = means[comp] + 0.05 * rng.standard_normal((n, 3))
    elif cfg.idx == 5:
        x = rng.random((n, 2))
    else:  # pragma: no cover
        raise ValueError(cfg.idx)
    return np.ascontiguousarray(x, dtype=np.float64)


def config_queries(cfg: Config) -> np.ndarray:
    """Query points z (M x d): U[0,1]^d, drawn after x from a separate stream."""
    rng = np.random.default_rng([cfg.idx - 1, 77])
    return np.ascontiguousarray(rng.random((cfg.m, cfg.d)))


def config_vector(cfg: Config, r: int = 0, n: int | None = None) -> np.ndarray:
    """The vector v of apply r: N(0,1) float64."""
    rng = np.random.default_rng([cfg.idx - 1, 1000 + r])
    return rng.standard_normal(cfg.n if n is None else n)


def config_response(cfg: Config, x: np.ndarray) -> np.ndarray:
    """Config 5 response: y = 1 + 0.5 x1 - 0.3 x2 + sin(6 x1) cos(4 x2) + N(0, sigma^2)."""
    rng = np.random.default_rng([cfg.idx - 1, 55])
    f = 1.0 + 0.5 * x[:, 0] - 0.3 * x[:, 1] + np.sin(6 * x[:, 0]) * np.cos(4 * x[:, 1])
    return f + cfg.noise_sigma * rng.standard_normal(x.shape[0])


def sample_rows(x: np.ndarray, count: int = 2048, seed: int = 12345) -> np.ndarray:
    """Seeded rows to check at large N: random rows plus the
    argmin/argmax row of each coordinate (boundary rows).  Sorted, unique, int64."""
    n, d = x.shape
    if count >= n:
        return np.arange(n, dtype=np.int64)
    extra = set()
    for k in range(d):
        extra.add(int(np.argmin(x[:, k])))
        extra.add(int(np.argmax(x[:, k])))
    rng = np.random.default_rng(seed)
    rows = set(int(i) for i in rng.choice(n, count - len(extra), replace=False))
    rows |= extra
    return np.array(sorted(rows), dtype=np.int64)
