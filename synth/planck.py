"""Group-integrated Planck function — INPUT GENERATION ONLY.

Used to build the emission sources q_g = (sigma_g + 1/(c dt)) B_g(T) and the
inflow B_g(T_bdr) of configs C2/C4/C5 (BASELINE.json:8-11).  Both the oracle and
the CUDA path receive the resulting bytes; neither evaluates Planck itself.

PAPER.md:106-125 (eq:planck, eq:black_body): B_g(T) = B(T) b_g(T) with
B(T) = a c T^4 and b_g(T) = (15/pi^4) int_{nu_g/T}^{nu_{g+1}/T} x^3/(e^x-1) dx,
"computed using polylogarithmic and Taylor series expansions" (Clark).
Reading R14: a = c = 1; the missing spectral tail is not renormalised.
"""
from __future__ import annotations

import math

import numpy as np

# Bernoulli numbers B_k (B_1 = -1/2 convention) for t/(e^t-1) = sum B_k t^k / k!
_BERN = {
    0: 1.0, 1: -0.5, 2: 1.0 / 6.0, 4: -1.0 / 30.0, 6: 1.0 / 42.0, 8: -1.0 / 30.0,
    10: 5.0 / 66.0, 12: -691.0 / 2730.0, 14: 7.0 / 6.0, 16: -3617.0 / 510.0,
    18: 43867.0 / 798.0, 20: -174611.0 / 330.0, 22: 854513.0 / 138.0,
    24: -236364091.0 / 2730.0, 26: 8553103.0 / 6.0,
}
_PI4_15 = math.pi ** 4 / 15.0


def _int_small(x: np.ndarray) -> np.ndarray:
    """int_0^x t^3/(e^t-1) dt = sum_k B_k x^(k+3) / (k! (k+3)), |x| < 2 pi."""
    out = np.zeros_like(x)
    for k, bk in _BERN.items():
        out += bk * x ** (k + 3) / (math.factorial(k) * (k + 3))
    return out


def _int_large(x: np.ndarray) -> np.ndarray:
    """int_0^x t^3/(e^t-1) dt = pi^4/15 - sum_n e^{-n x}(x^3/n + 3x^2/n^2 + 6x/n^3 + 6/n^4)."""
    tail = np.zeros_like(x)
    for n in range(1, 40):
        tail += np.exp(-n * x) * (x ** 3 / n + 3 * x ** 2 / n ** 2 + 6 * x / n ** 3 + 6 / n ** 4)
    return _PI4_15 - tail


def planck_cdf(x) -> np.ndarray:
    """P(x) = (15/pi^4) int_0^x t^3/(e^t-1) dt, P(inf) = 1."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    small = x < 2.0
    out[small] = _int_small(x[small])
    big = ~small
    xb = np.minimum(x[big], 700.0)
    out[big] = _int_large(xb)
    return out / _PI4_15


def group_bounds(G: int, lo: float = 0.01, hi: float = 100.0) -> np.ndarray:
    """Log-spaced bounds nu_g = lo * (hi/lo)^(g/G), g = 0..G."""
    return lo * (hi / lo) ** (np.arange(G + 1) / G)


def group_energy(bounds: np.ndarray) -> np.ndarray:
    """Reading R8: E_g = sqrt(nu_g nu_{g+1}) (geometric group centre)."""
    return np.sqrt(bounds[:-1] * bounds[1:])


def planck_groups(T, bounds: np.ndarray) -> np.ndarray:
    """B_g(T) = T^4 [P(nu_{g+1}/T) - P(nu_g/T)], a = c = 1.  Shape T.shape + (G,)."""
    T = np.asarray(T, dtype=np.float64)
    x = bounds[None, :] / T.reshape(-1, 1)
    P = planck_cdf(x)
    B = (T.reshape(-1, 1) ** 4) * (P[:, 1:] - P[:, :-1])
    return B.reshape(T.shape + (len(bounds) - 1,))
