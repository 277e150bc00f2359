"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no Gram products, no monomial
ranking, no coefficient expansion).  It only draws seeded random numbers with
the shapes and distributions of BASELINE.json's configs, and states those
configs.  Both sides (the fp64 oracle and the CUDA path) compute their own
targets from the same drawn factors, e.g. the planted target p = coef(W W^T)
is computed by each side from W.

Recipe:
  * V0 : N x r, iid N(0, 1/N)            (BASELINE.json configs, "V init iid N(0,1/N)")
  * W  : N x r*, iid N(0, 1/N)           (planted SOS factor, "w_k iid N(0,1/N)")
  * residual probes: iid N(0, 1) vectors of length M (used only to exercise the
    backward in isolation; any vector is a valid residual)
Every draw uses numpy's PCG64 seeded through SeedSequence(seed, spawn_key=(stream,)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# stream ids (spawn keys) so that V0, W and probes never share random numbers
STREAM_V0 = 1
STREAM_W = 2
STREAM_PROBE = 3
STREAM_POINTS = 4


@dataclass(frozen=True)
class Config:
    name: str
    n: int          # variables
    d: int          # half degree; the form has degree 2d
    r: int          # number of squares (columns of V)
    r_star: int     # planted rank
    eps: float = 0.0  # weight of eps*(sum x_i^2)^(2d/2) added to the target (config 3)

    @property
    def N(self) -> int:
        return math.comb(self.n + self.d - 1, self.d)

    @property
    def M(self) -> int:
        return math.comb(self.n + 2 * self.d - 1, 2 * self.d)


# BASELINE.json "configs", in order.
CONFIGS = {
    "c0_n4_2d6": Config("c0_n4_2d6", n=4, d=3, r=20, r_star=10),
    "c1_n8_2d8": Config("c1_n8_2d8", n=8, d=4, r=330, r_star=165),
    "c2_n10_2d10": Config("c2_n10_2d10", n=10, d=5, r=2002, r_star=1001),
    "c2b_n10_2d10_r4004": Config("c2b_n10_2d10_r4004", n=10, d=5, r=4004, r_star=1001),
    "c3_n12_2d12": Config("c3_n12_2d12", n=12, d=6, r=12376, r_star=6188, eps=1e-3),
    "c4_n17_2d10": Config("c4_n17_2d10", n=17, d=5, r=20349, r_star=10175),
}
BENCH_CONFIG = "c4_n17_2d10"

# The paper's own timing table: random SOS quartics (2d = 4)
# in n = 10 ... 100 variables, full-rank over-parameterised factor.  Used only
# as context next to its quoted laptop timings (tools/paper_table.py); the
# planted target follows the recipe above (r* = N/2 Gaussian squares).
PAPER_QUARTICS = {
    f"q_n{n}": Config(f"q_n{n}", n=n, d=2, r=math.comb(n + 1, 2), r_star=math.comb(n + 1, 2) // 2)
    for n in (10, 15, 20, 25, 30, 100)
}
# seconds the paper reports for "our approach" on an Intel i7-6500U laptop
PAPER_QUARTIC_SECONDS = {"q_n10": 32.7, "q_n15": 46.0, "q_n20": 89.0, "q_n25": 234.0, "q_n30": 542.0,
                         "q_n100": 151000.0}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(seed, spawn_key=(stream,))))


def gaussian(rows: int, cols: int, std: float, seed: int, stream: int) -> np.ndarray:
    """rows x cols float32, iid N(0, std^2)."""
    g = _rng(seed, stream).standard_normal((rows, cols), dtype=np.float32)
    if std != 1.0:
        g *= np.float32(std)
    return g


def v0(N: int, r: int, seed: int = 0) -> np.ndarray:
    """Initial factor V0 ~ N(0, 1/N), N x r float32."""
    return gaussian(N, r, 1.0 / math.sqrt(N), seed, STREAM_V0)


def planted_w(N: int, r_star: int, seed: int = 0) -> np.ndarray:
    """Planted factor W ~ N(0, 1/N), N x r* float32; the target is coef(W W^T)."""
    return gaussian(N, r_star, 1.0 / math.sqrt(N), seed, STREAM_W)


def residual_probe(M: int, seed: int = 0) -> np.ndarray:
    """A seeded N(0,1) vector of length M used as a residual input."""
    return _rng(seed, STREAM_PROBE).standard_normal(M, dtype=np.float32)


def sphere_power_coefficients(beta: np.ndarray, d: int) -> np.ndarray:
    """Coefficients of (x_1^2 + ... + x_n^2)^d on the degree-2d basis whose
    exponent table is `beta` (M x n, any order): the multinomial d!/prod(g_v!)
    on beta = 2g, zero elsewhere.  BASELINE.json config 3 adds eps times this
    form to the planted target for strict positivity.  Pure target
    construction (multinomial theorem); no Gram or ranking arithmetic."""
    beta = np.asarray(beta, dtype=np.int64)
    even = np.all(beta % 2 == 0, axis=1)
    g = beta // 2
    lf = np.array([math.lgamma(k + 1) for k in range(d + 1)])
    out = np.zeros(beta.shape[0], dtype=np.float64)
    ge = g[even]
    out[even] = np.rint(np.exp(lf[d] - lf[ge].sum(axis=1)))
    return out


def points(count: int, n: int, seed: int = 0) -> np.ndarray:
    """Random evaluation points x in R^n (float64, N(0,1))."""
    return _rng(seed, STREAM_POINTS).standard_normal((count, n))
