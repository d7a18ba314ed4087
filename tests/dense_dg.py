"""Independent pin for the oracle: the GLOBAL lumped upwind-DG system assembled
in the paper's jump/average form and solved densely (tiny meshes only).

This is a second formulation, written from PAPER.md directly and sharing no
code with oracle/sweep_oracle.c:
  * interior faces use eq:upwind,
        Omega.n psi^ = Omega.n {psi} + |Omega.n|/2 [[psi]],
    tested against [[u]] as in eq:dgsn_transport;
  * boundary faces use the boundary flux PAPER.md:321-326;
  * all integrals use the tensor Gauss-Lobatto rule (reading R1
    for p = 2), and the derivative matrix is obtained from a Vandermonde
    inverse (numpy), not from the Lagrange-product formula the oracle uses.
The unknowns of ALL elements are solved at once, so no sweep ordering enters.
"""
from __future__ import annotations

import numpy as np


def _gll(p: int):
    if p == 1:
        return np.array([0.0, 1.0]), np.array([0.5, 0.5])
    if p == 2:
        return np.array([0.0, 0.5, 1.0]), np.array([1.0, 4.0, 1.0]) / 6.0
    raise ValueError(p)


def _dmat(xi: np.ndarray) -> np.ndarray:
    """Dm[a, b] = d l_b / dxi at xi_a, via the monomial Vandermonde matrix."""
    m = len(xi)
    V = np.vander(xi, m, increasing=True)          # V[a, c] = xi_a^c
    C = np.linalg.inv(V)                            # l_b(x) = sum_c C[c, b] x^c
    dV = np.zeros_like(V)
    for c in range(1, m):
        dV[:, c] = c * xi ** (c - 1)
    return dV @ C


def assemble_global(prob, d: int, g: int):
    """(A, b) of the global system for (d, g), unknowns ordered (element, node)."""
    dim, p = prob.dim, prob.p
    nx = prob.nx
    ny = prob.ny if dim == 2 else 1
    np1 = p + 1
    n = np1 ** dim
    xi, wh = _gll(p)
    Dm = _dmat(xi)
    hx = prob.lx / nx
    hy = prob.ly / ny if dim == 2 else 1.0
    ox = prob.omega[d, 0]
    oy = prob.omega[d, 1] if dim == 2 else 0.0
    G = prob.sigma.shape[1]
    N = nx * ny * n
    A = np.zeros((N, N))
    b = np.zeros(N)

    def node_ab(k):
        return (k % np1, k // np1) if dim == 2 else (k, 0)

    def gid(i, j, k):
        return (i + nx * j) * n + k

    def vol_w(k):
        a, bb = node_ab(k)
        return hx * hy * wh[a] * wh[bb] if dim == 2 else hx * wh[a]

    # volume terms: -int Omega.grad(u) psi + int sigma~ u psi = int u q
    for j in range(ny):
        for i in range(nx):
            e = i + nx * j
            st = prob.sigma[e, g] + prob.inv_c_dt
            for k in range(n):
                ak, bk = node_ab(k)
                A[gid(i, j, k), gid(i, j, k)] += st * vol_w(k)
                b[gid(i, j, k)] += vol_w(k) * prob.q[e, k, g]
                for l in range(n):
                    al, bl = node_ab(l)
                    dx = Dm[al, ak] / hx if bl == bk else 0.0
                    dy = (Dm[bl, bk] / hy if al == ak else 0.0) if dim == 2 else 0.0
                    A[gid(i, j, k), gid(i, j, l)] -= vol_w(l) * (ox * dx + oy * dy)

    # faces as lists of (K1 node gid, K2 node gid or None, face weight, Omega.n, bnode index)
    faces = []
    if dim == 1:
        for i in range(nx - 1):
            faces.append((gid(i, 0, p), gid(i + 1, 0, 0), 1.0, ox, None))
        faces.append((gid(nx - 1, 0, p), None, 1.0, ox, 1))   # x = 1, n = +x
        faces.append((gid(0, 0, 0), None, 1.0, -ox, 0))       # x = 0, n = -x
    else:
        for j in range(ny):
            for bb in range(np1):
                wf = hy * wh[bb]
                for i in range(nx - 1):
                    faces.append((gid(i, j, p + np1 * bb), gid(i + 1, j, 0 + np1 * bb), wf, ox, None))
                faces.append((gid(0, j, 0 + np1 * bb), None, wf, -ox, j * np1 + bb))
                faces.append((gid(nx - 1, j, p + np1 * bb), None, wf, ox, ny * np1 + j * np1 + bb))
        for i in range(nx):
            for a in range(np1):
                wf = hx * wh[a]
                for j in range(ny - 1):
                    faces.append((gid(i, j, a + np1 * p), gid(i, j + 1, a), wf, oy, None))
                faces.append((gid(i, 0, a), None, wf, -oy, 2 * ny * np1 + i * np1 + a))
                faces.append((gid(i, ny - 1, a + np1 * p), None, wf, oy, 2 * ny * np1 + nx * np1 + i * np1 + a))

    for (k1, k2, wf, on, bn) in faces:
        if k2 is not None:
            # int Omega.n [[u]] {psi} + 1/2 int |Omega.n| [[u]] [[psi]]
            c1 = wf * (0.5 * on + 0.5 * abs(on))   # coefficient of psi_1
            c2 = wf * (0.5 * on - 0.5 * abs(on))   # coefficient of psi_2
            A[k1, k1] += c1
            A[k1, k2] += c2
            A[k2, k1] -= c1
            A[k2, k2] -= c2
        else:
            if on > 0:
                A[k1, k1] += wf * on                          # Gamma_b^+: Omega.n u psi
            elif on < 0:
                b[k1] -= wf * on * prob.inflow[bn, g]        # - int_{Gamma_b^-} Omega.n u psi_in
    return A, b


def solve_global(prob, d: int, g: int) -> np.ndarray:
    """psi_{d,g} [N_el][n] from one dense solve of the assembled global system."""
    A, b = assemble_global(prob, d, g)
    nel = prob.nx * (prob.ny if prob.dim == 2 else 1)
    return np.linalg.solve(A, b).reshape(nel, -1)


def element_weights(prob) -> np.ndarray:
    """Lumped mass weights W_k of one element (tensor GLL)."""
    _, wh = _gll(prob.p)
    hx = prob.lx / prob.nx
    if prob.dim == 1:
        return hx * wh
    hy = prob.ly / prob.ny
    return hx * hy * np.outer(wh, wh).reshape(-1)   # k = a + (p+1) b  ->  wh[b] * wh[a]


def zero_and_scale(x: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Zero-and-scale fixup (SPEC.md's fixup_zero_and_scale): negatives to
    0, the rest scaled so sum W x is kept; a non-positive sum zeroes the element."""
    if (x >= 0).all():
        return x
    total = float(W @ x)
    if total <= 0:
        return np.zeros_like(x)
    pos = np.where(x > 0, x, 0.0)
    return pos * (total / float(W @ pos))


def sweep_blocks(prob, d: int, g: int, fixup: bool = True) -> np.ndarray:
    """Element-by-element block forward substitution of the global system in upwind
    order, with the fixup applied to each element before its downwind neighbours use
    it (the sweep of PAPER.md:987 written on the jump/average assembly)."""
    A, b = assemble_global(prob, d, g)
    nx = prob.nx
    ny = prob.ny if prob.dim == 2 else 1
    n = A.shape[0] // (nx * ny)
    ox = prob.omega[d, 0]
    oy = prob.omega[d, 1] if prob.dim == 2 else 0.0
    W = element_weights(prob)
    psi = np.zeros(A.shape[0])
    jr = range(ny) if oy >= 0 else range(ny - 1, -1, -1)
    for j in jr:
        ir = range(nx) if ox >= 0 else range(nx - 1, -1, -1)
        for i in ir:
            e = i + nx * j
            sl = slice(e * n, (e + 1) * n)
            r = b[sl] - A[sl, :] @ psi + A[sl, sl] @ psi[sl]
            x = np.linalg.solve(A[sl, sl], r)
            psi[sl] = zero_and_scale(x, W) if fixup else x
    return psi.reshape(nx * ny, n)
