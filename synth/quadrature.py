"""Angular quadrature sets — INPUT DATA shared by the oracle and the CUDA path.

This module only builds the direction set {Omega_d, w_d} that the paper's
problem statement takes as input ("a set of discrete directions
taken from a quadrature rule for the unit sphere, {Omega_d, w_d}").  It holds
none of the method's arithmetic (no alpha, no closure coefficients, no sweep).

Readings:
  * normalisation sum_d w_d = 1 (BASELINE.json configs "weights normalised to
    sum 1");
  * 1-D sets are Gauss-Legendre S_N in mu, stored as omega[d] = (mu, 0, 0);
  * 2-D sets are products of Gauss-Legendre polar nodes xi and equispaced
    azimuths omega_k = (k + 1/2) 2 pi / N_az, so no direction has
    Omega_x = 0 or Omega_y = 0.

Nodes are built with exact +-symmetry (positive roots mirrored) and the
azimuths with exact 90-degree rotational symmetry (first quadrant rotated), so
that +-Omega_z pairs share bit-identical (Omega_x, Omega_y).
"""
from __future__ import annotations

import math

import numpy as np


def gauss_legendre(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Legendre nodes/weights on (-1, 1), sum w = 2, ascending nodes.

    Newton iteration on P_n with the three-term recurrence; only the positive
    roots are iterated and the negative ones are their exact mirror images.
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    xs = []
    ws = []
    m = n // 2
    for i in range(m):
        # Chebyshev-like initial guess for the i-th largest root
        x = math.cos(math.pi * (i + 0.75) / (n + 0.5))
        for _ in range(100):
            p0, p1 = 1.0, x
            for k in range(2, n + 1):
                p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
            dp = n * (x * p1 - p0) / (x * x - 1.0)
            dx = p1 / dp
            x -= dx
            if abs(dx) < 1e-17:
                break
        p0, p1 = 1.0, x
        for k in range(2, n + 1):
            p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        dp = n * (x * p1 - p0) / (x * x - 1.0)
        xs.append(x)
        ws.append(2.0 / ((1.0 - x * x) * dp * dp))
    pos_x = np.array(xs[::-1])
    pos_w = np.array(ws[::-1])
    if n % 2 == 1:
        # middle root x = 0
        p0, p1 = 1.0, 0.0
        for k in range(2, n + 1):
            p0, p1 = p1, ((2 * k - 1) * 0.0 * p1 - (k - 1) * p0) / k
        dp = n * (0.0 * p1 - p0) / (-1.0)
        mid_w = 2.0 / (dp * dp)
        x = np.concatenate([-pos_x[::-1], [0.0], pos_x])
        w = np.concatenate([pos_w[::-1], [mid_w], pos_w])
    else:
        x = np.concatenate([-pos_x[::-1], pos_x])
        w = np.concatenate([pos_w[::-1], pos_w])
    return x, w


def slab_set(n: int) -> tuple[np.ndarray, np.ndarray]:
    """1-D Gauss-Legendre S_n set: omega [n][3] with omega[d,0] = mu_d, w summing to 1."""
    mu, w = gauss_legendre(n)
    w = w / w.sum()
    om = np.zeros((n, 3))
    om[:, 0] = mu
    return om, w


def product_set(n_polar: int, n_az: int) -> tuple[np.ndarray, np.ndarray]:
    """2-D product set: GL(n_polar) in xi = Omega_z times n_az equispaced azimuths.

    Omega = (sqrt(1-xi^2) cos w_k, sqrt(1-xi^2) sin w_k, xi),
    w_k = (k + 1/2) 2 pi / n_az, weight = (w_GL / 2) / n_az.  Direction index
    d = i_polar * n_az + k.  n_az must be a multiple of 4 (exact rotation).
    """
    if n_az % 4 != 0:
        raise ValueError("n_az must be a multiple of 4")
    xi, wxi = gauss_legendre(n_polar)
    q = n_az // 4
    c1 = np.array([math.cos((k + 0.5) * 2.0 * math.pi / n_az) for k in range(q)])
    s1 = np.array([math.sin((k + 0.5) * 2.0 * math.pi / n_az) for k in range(q)])
    # rotate the first quadrant by 90 degrees three times: (c, s) -> (-s, c)
    cs = [c1]
    ss = [s1]
    for _ in range(3):
        c_prev, s_prev = cs[-1], ss[-1]
        cs.append(-s_prev)
        ss.append(c_prev.copy())
    cos_az = np.concatenate(cs)
    sin_az = np.concatenate(ss)
    om = np.zeros((n_polar * n_az, 3))
    w = np.zeros(n_polar * n_az)
    for ip in range(n_polar):
        st = math.sqrt(1.0 - xi[ip] * xi[ip])
        for k in range(n_az):
            d = ip * n_az + k
            om[d, 0] = st * cos_az[k]
            om[d, 1] = st * sin_az[k]
            om[d, 2] = xi[ip]
            w[d] = 0.5 * wxi[ip] / n_az
    # exact +-xi symmetry of sqrt(1-xi^2): the node set is mirrored, so the
    # (Omega_x, Omega_y) of +-xi pairs are bit-identical by construction.
    w = w / w.sum()
    return om, w
