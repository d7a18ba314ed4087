"""Pins for the CPU oracle (-m "not gpu"): each checks the oracle against
something other than itself — closed forms, an independent global assembly,
invariants the paper fixes, symmetries, convergence, and derived fixtures.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from synth.configs import Problem, bnode_index, random_problem
from tests.dense_dg import solve_global

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- quadrature
@pytest.mark.parametrize("N", [2, 4, 8, 16])
def test_slab_moment_identities(N):
    """sum w mu^k = 1/(k+1) (k even), 0 (k odd), k <= 2N-1 (Gauss exactness); sum w = 1 (R3)."""
    om, w = synth.slab_set(N)
    mu = om[:, 0]
    for k in range(2 * N):
        exact = 1.0 / (k + 1) if k % 2 == 0 else 0.0
        assert abs(np.sum(w * mu ** k) - exact) < 2e-15


@pytest.mark.parametrize("npol,naz", [(4, 16), (8, 16), (2, 8)])
def test_product_set_identities(npol, naz):
    """sum w = 1, sum w Omega = 0, sum w Omega Omega = I/3 (north_star)."""
    om, w = synth.product_set(npol, naz)
    assert abs(w.sum() - 1.0) < 1e-15
    assert np.abs(w @ om).max() < 1e-15
    M = (om * w[:, None]).T @ om
    assert np.abs(M - np.eye(3) / 3.0).max() < 1e-15
    assert np.abs(np.linalg.norm(om, axis=1) - 1.0).max() < 1e-15


def test_alpha_closed_forms():
    """eq:alpha: S2 -> 1/sqrt(3) exactly; -> 1/2 as N grows; scale invariant."""
    om, w = synth.slab_set(2)
    P = Problem("a", 1, 1, 1, 1, om, w, np.ones((1, 1)), np.ones((1, 2, 1)), np.zeros((2, 1)), 0.0)
    assert abs(oracle.alpha(P)[0] - 1.0 / math.sqrt(3.0)) < 1e-15
    prev = 1.0
    for N in (4, 8, 16, 64):
        om, w = synth.slab_set(N)
        P.omega, P.w = om, w
        a = oracle.alpha(P)[0]
        assert 0.5 < a < prev
        prev = a
    assert abs(prev - 0.5) < 2e-4
    P.w = 3.0 * P.w
    assert abs(oracle.alpha(P)[0] - prev) < 1e-15


# ---------------------------------------------------------- golden fixtures
def test_golden_g1_slab():
    gd = json.load(open(os.path.join(GOLD, "g1_slab.json")))
    om, w = synth.slab_set(4)
    P = Problem("g1", 1, 4, 1, 1, om, w, np.array(gd["sigma_tilde"])[:, None], np.ones((4, 2, 1)),
                np.array([[1.0], [0.0]]), 0.0)
    f = oracle.unpack(oracle.sweep(P), 1, 4, 1, 1)
    assert abs(oracle.alpha(P)[0] - gd["alpha"]) < 1e-15
    for key, got in (("phi", f["phi"].ravel()), ("J", f["J"].ravel()), ("Txx", f["T"].ravel()),
                     ("beta", f["beta"]), ("Jplus", f["Jplus"])):
        assert np.abs(got - np.array(gd[key])).max() < 1e-13, key


@pytest.mark.parametrize("p", [1, 2])
def test_golden_g2_square(p):
    gd = json.load(open(os.path.join(GOLD, "g2_square.json")))
    om, w = synth.product_set(4, 16)
    n = (p + 1) ** 2
    fl = np.zeros((2 * 4 * (p + 1), 1))
    fl[: 2 * (p + 1)] = 1.0
    P = Problem("g2", 2, 2, 2, p, om, w, np.array(gd["sigma_tilde"])[:, None], np.ones((4, n, 1)), fl, 0.0)
    f = oracle.unpack(oracle.sweep(P), 2, 2, 2, p)
    sums = gd[f"p{p}_sums"]
    scale = sums["phi"]
    got = {"phi": f["phi"].sum(), "Jx": f["J"][0].sum(), "Jy": f["J"][1].sum(),
           "Txx": f["T"][0].sum(), "Txy": f["T"][1].sum(), "Tyy": f["T"][2].sum()}
    for k, v in sums.items():
        assert abs(got[k] - v) < 1e-14 * scale, k
    if p == 1:
        assert np.abs(f["phi"][0] - np.array(gd["p1_phi_e00"])).max() < 1e-14


# ------------------------------------------------- closed-form transmission
@pytest.mark.parametrize("mu_sign", [1, -1])
def test_slab_p1_transmission_closed_form(mu_sign):
    """1-D p=1 pure absorber, uniform sigma~ (derived by hand from the
    2x2 element system): with c = |mu|/h, tau = sigma~/c,
        psi_out = t psi_in, t = 1/(1 + tau + tau^2/2), psi_in-node = (1+tau) psi_out,
    so the outflow node of the i-th cell downstream is t^(i+1) psi_in."""
    nx, st, mu = 12, 3.7, 0.41 * mu_sign
    om = np.array([[mu, 0.0, 0.0]])
    w = np.array([1.0])
    fl = np.zeros((2, 1))
    fl[0 if mu > 0 else 1, 0] = 2.5
    P = Problem("t", 1, nx, 1, 1, om, w, np.full((nx, 1), st), np.zeros((nx, 2, 1)), fl, 0.0)
    psi = oracle.sweep_psi(P, 0, 0)
    tau = st * (1.0 / nx) / abs(mu)
    t = 1.0 / (1.0 + tau + 0.5 * tau * tau)
    for ii in range(nx):
        i = ii if mu > 0 else nx - 1 - ii
        out_node, in_node = (1, 0) if mu > 0 else (0, 1)
        assert abs(psi[i, out_node] - 2.5 * t ** (ii + 1)) < 1e-14 * 2.5
        assert abs(psi[i, in_node] - 2.5 * (1 + tau) * t ** (ii + 1)) < 1e-14 * 2.5


# --------------------------------------------- global dense solve equality
CASES = [
    (1, 5, 1, 1, 4, 2), (1, 6, 1, 2, 5, 2), (2, 3, 4, 1, 6, 2), (2, 4, 3, 2, 6, 2),
    (2, 1, 1, 2, 4, 1), (2, 2, 5, 1, 5, 3), (2, 5, 2, 2, 3, 2),
]


@pytest.mark.parametrize("dim,nx,ny,p,ndir,G", CASES)
def test_sweep_equals_dense_global_solve(dim, nx, ny, p, ndir, G):
    """The sweep reaches exactly the solution of the global system."""
    prob = random_problem(7 * nx + 13 * ny + p, dim, nx, ny, p, ndir, G)
    for d in range(ndir):
        for g in range(G):
            ref = solve_global(prob, d, g)
            got = oracle.sweep_psi(prob, d, g)
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (d, g)


def test_dense_covers_all_quadrants():
    """The random direction sets used above really hit all 4 quadrants."""
    seen = set()
    for (dim, nx, ny, p, ndir, G) in CASES:
        if dim != 2:
            continue
        prob = random_problem(7 * nx + 13 * ny + p, dim, nx, ny, p, ndir, G)
        seen |= {(np.sign(o[0]), np.sign(o[1])) for o in prob.omega}
    assert len(seen) == 4


# ------------------------------------------------ moments from psi (definition)
def test_moments_match_definition_from_psi():
    """Gray moments = weighted sums of the oracle's psi."""
    prob = random_problem(3, 2, 3, 2, 2, 5, 2)
    out = oracle.unpack(oracle.sweep(prob), 2, 3, 2, 2)
    phi = np.zeros_like(out["phi"])
    J = np.zeros_like(out["J"])
    T = np.zeros_like(out["T"])
    for d in range(prob.n_dir):
        o = prob.omega[d]
        for g in range(prob.G):
            psi = solve_global(prob, d, g)  # independent psi
            wd = prob.w[d]
            phi += wd * psi
            J[0] += wd * o[0] * psi
            J[1] += wd * o[1] * psi
            T[0] += wd * (o[0] ** 2 - 1 / 3) * psi
            T[1] += wd * o[0] * o[1] * psi
            T[2] += wd * (o[1] ** 2 - 1 / 3) * psi
    for a, b in ((phi, out["phi"]), (J, out["J"]), (T, out["T"])):
        assert np.abs(a - b).max() < 1e-13 * np.abs(phi).max()


# ------------------------------------------- infinite-medium constant solution
@pytest.mark.parametrize("dim,p", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_constant_solution_exact(dim, p):
    """q = sigma~ Q and inflow Q on every face => psi == Q (north_star 'DG exactness
    for a spatially constant solution'), so phi = Q, J = 0, T = 0 (sum w Omega
    Omega = I/3), beta = 0 (definition of alpha), J+ = Q sum_{Omega.n>0} w Omega.n."""
    nx, ny = (7, 1) if dim == 1 else (5, 4)
    om, w = synth.slab_set(8) if dim == 1 else synth.product_set(4, 16)
    G = 2
    rng = np.random.default_rng(5)
    n = (p + 1) ** dim
    ne = nx * ny
    sig = rng.uniform(0.1, 100.0, size=(ne, G))
    Q = np.array([1.7, 0.3])
    inv = 0.5
    q = np.broadcast_to(((sig + inv) * Q[None, :])[:, None, :], (ne, n, G)).copy()
    nb = 2 if dim == 1 else 2 * (nx + ny) * (p + 1)
    fl = np.broadcast_to(Q[None, :], (nb, G)).copy()
    P = Problem("c", dim, nx, ny, p, om, w, sig, q, fl, inv)
    f = oracle.unpack(oracle.sweep(P), dim, nx, ny, p)
    Qs = Q.sum()
    assert np.abs(f["phi"] - Qs).max() < 1e-13 * Qs
    assert np.abs(f["J"]).max() < 1e-13 * Qs
    assert np.abs(f["T"]).max() < 1e-13 * Qs
    assert np.abs(f["beta"]).max() < 1e-13 * Qs
    a = oracle.alpha(P)
    if dim == 2:
        # J+ = Q * sum_{Omega.n > 0} w Omega.n = Q * alpha_n / 2 ... check directly
        jp_x = Qs * np.sum(w * np.maximum(om[:, 0], 0.0))
        assert abs(f["Jplus"][0] - Qs * np.sum(w * np.maximum(-om[:, 0], 0.0))) < 1e-13 * Qs
        assert abs(f["Jplus"][bnode_index("x+", 0, 0, nx, ny, p)] - jp_x) < 1e-13 * Qs
        # for a symmetric set, J+ = alpha/2 * phi
        assert abs(jp_x - 0.5 * a[1] * Qs) < 1e-13 * Qs


# -------------------------------------------------------- particle balance
@pytest.mark.parametrize("dim,p", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_global_particle_balance_gray(dim, p):
    """Testing the weak form with u == 1 (sum_k l_k = 1): interior face terms cancel
    and the streaming volume term vanishes, leaving, for G = 1,
      sum_e sum_k W_k (q_k - sigma~ phi_k) = sum_bnodes W^f (J+ + J_in),
    J_in = sum_{Omega.n<0} w (Omega.n) psi_in.  Pins phi and J+ jointly."""
    nx, ny = (9, 1) if dim == 1 else (4, 5)
    prob = random_problem(11, dim, nx, ny, p, 6 if dim == 2 else 4, 1)
    f = oracle.unpack(oracle.sweep(prob), dim, nx, ny, p)
    np1 = p + 1
    xi_w = {1: np.array([0.5, 0.5]), 2: np.array([1, 4, 1]) / 6.0}[p]
    hx = 1.0 / nx
    hy = 1.0 / ny if dim == 2 else 1.0
    if dim == 1:
        W = hx * xi_w
    else:
        W = hx * hy * np.array([xi_w[k % np1] * xi_w[k // np1] for k in range(np1 * np1)])
    st = prob.sigma[:, 0] + prob.inv_c_dt
    lhs = np.sum(W[None, :] * (prob.q[:, :, 0] - st[:, None] * f["phi"]))
    # boundary: face weights and normals per boundary node
    om, w = prob.omega, prob.w
    rhs = 0.0
    nb = f["beta"].size
    for t in range(nb):
        if dim == 1:
            wf, nvec = 1.0, (-1.0 if t == 0 else 1.0)
            on = om[:, 0] * nvec
        else:
            if t < 2 * ny * np1:
                node = t % np1
                wf = hy * xi_w[node]
                on = -om[:, 0] if t < ny * np1 else om[:, 0]
            else:
                node = (t - 2 * ny * np1) % np1
                wf = hx * xi_w[node]
                on = -om[:, 1] if t < 2 * ny * np1 + nx * np1 else om[:, 1]
        jin = np.sum(w * np.minimum(on, 0.0)) * prob.inflow[t, 0]
        rhs += wf * (f["Jplus"][t] + jin)
    assert abs(lhs - rhs) < 1e-12 * max(abs(lhs), np.abs(prob.q).max())


def test_per_direction_balance():
    """Per (d,g): sum W (q - sigma~ psi) = sum_bnodes W^f (Omega.n) psi^ (upwind psi^)."""
    prob = random_problem(12, 2, 5, 3, 2, 4, 2)
    np1 = 3
    xi_w = np.array([1, 4, 1]) / 6.0
    hx, hy = 1 / 5, 1 / 3
    W = hx * hy * np.array([xi_w[k % np1] * xi_w[k // np1] for k in range(9)])
    for d in range(4):
        for g in range(2):
            psi = oracle.sweep_psi(prob, d, g)
            st = prob.sigma[:, g] + prob.inv_c_dt
            lhs = np.sum(W[None, :] * (prob.q[:, :, g] - st[:, None] * psi))
            ox, oy = prob.omega[d, :2]
            rhs = 0.0
            for j in range(3):
                for b in range(np1):
                    wf = hy * xi_w[b]
                    for face, on, e, k in (("x-", -ox, 0 + 5 * j, 0 + np1 * b), ("x+", ox, 4 + 5 * j, 2 + np1 * b)):
                        val = psi[e, k] if on > 0 else prob.inflow[bnode_index(face, j, b, 5, 3, 2), g]
                        rhs += wf * on * val
            for i in range(5):
                for a in range(np1):
                    wf = hx * xi_w[a]
                    for face, on, e, k in (("y-", -oy, i, a), ("y+", oy, i + 5 * 2, a + np1 * 2)):
                        val = psi[e, k] if on > 0 else prob.inflow[bnode_index(face, i, a, 5, 3, 2), g]
                        rhs += wf * on * val
            assert abs(lhs - rhs) < 1e-12 * np.abs(prob.q).max()


# ------------------------------------------------------------ convergence
def test_slab_pure_absorber_convergence():
    """1-D: psi(1) -> psi_in exp(-sigma~/mu) at O(h^2) for p = 1 (north_star)."""
    st, mu = 2.0, 0.6
    exact = math.exp(-st / mu)
    errs = []
    for nx in (8, 16, 32, 64):
        P = Problem("cv", 1, nx, 1, 1, np.array([[mu, 0, 0]]), np.array([1.0]), np.full((nx, 1), st),
                    np.zeros((nx, 2, 1)), np.array([[1.0], [0.0]]), 0.0)
        errs.append(abs(oracle.sweep_psi(P, 0, 0)[-1, 1] - exact))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(r > 1.8 for r in rates), rates


def _l2_error_2d(prob, psi, exact_fn):
    """L2 error with a 3-point Gauss-Legendre tensor rule per element."""
    gx, gw = np.polynomial.legendre.leggauss(3)
    gx = 0.5 * (gx + 1.0)
    gw = 0.5 * gw
    p = prob.p
    xi = {1: np.array([0.0, 1.0]), 2: np.array([0.0, 0.5, 1.0])}[p]

    def lag(t):
        L = np.ones((len(xi), len(t)))
        for a in range(len(xi)):
            for m in range(len(xi)):
                if m != a:
                    L[a] *= (t - xi[m]) / (xi[a] - xi[m])
        return L

    La = lag(gx)
    nx, ny = prob.nx, prob.ny
    hx, hy = 1.0 / nx, 1.0 / ny
    err2 = 0.0
    np1 = p + 1
    for j in range(ny):
        for i in range(nx):
            e = i + nx * j
            c = psi[e].reshape(np1, np1)  # [b][a]
            u = La.T @ c.T @ La            # u[qa, qb]
            X = (i + gx)[:, None] * hx
            Y = (j + gx)[None, :] * hy
            ex = exact_fn(X, Y)
            err2 += np.sum(gw[:, None] * gw[None, :] * (u - ex) ** 2) * hx * hy
    return math.sqrt(err2)


@pytest.mark.parametrize("p,min_rate", [(1, 1.7), (2, 2.7)])
def test_2d_pure_absorber_convergence(p, min_rate):
    """Smooth pure absorber psi = g(y - (Oy/Ox) x) exp(-sigma~ x / Ox) with exact
    nodal inflow on both inflow edges: L2 order ~ p+1 (north_star)."""
    ox, oy = 0.8, 0.45
    st = 1.5
    gfun = lambda s: 1.0 + 0.5 * np.sin(2.0 * s)  # noqa: E731
    exact = lambda X, Y: gfun(Y - (oy / ox) * X) * np.exp(-st * X / ox)  # noqa: E731
    errs = []
    for nx in (4, 8, 16):
        ny = nx
        n = (p + 1) ** 2
        nb = 2 * (nx + ny) * (p + 1)
        fl = np.zeros((nb, 1))
        xi = {1: [0.0, 1.0], 2: [0.0, 0.5, 1.0]}[p]
        for j in range(ny):
            for b in range(p + 1):
                y = (j + xi[b]) / ny
                fl[bnode_index("x-", j, b, nx, ny, p), 0] = exact(0.0, y)
        for i in range(nx):
            for a in range(p + 1):
                x = (i + xi[a]) / nx
                fl[bnode_index("y-", i, a, nx, ny, p), 0] = exact(x, 0.0)
        om = np.array([[ox, oy, math.sqrt(1 - ox * ox - oy * oy)]])
        P = Problem("cv2", 2, nx, ny, p, om, np.array([1.0]), np.full((nx * ny, 1), st),
                    np.zeros((nx * ny, n, 1)), fl, 0.0)
        errs.append(_l2_error_2d(P, oracle.sweep_psi(P, 0, 0), exact))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] > min_rate, rates


# ------------------------------------------------------------ symmetry
def _rotate90(prob):
    """Rotate a square problem by +90 deg about the centre: (x,y) -> (1-y, x),
    element (i,j) -> (N-1-j, i), node (a,b) -> (p-b, a), Omega -> (-Oy, Ox)."""
    N, p = prob.nx, prob.p
    np1 = p + 1
    n = np1 * np1
    sig = np.zeros_like(prob.sigma)
    q = np.zeros_like(prob.q)
    emap = np.zeros(N * N, dtype=int)
    kmap = np.zeros(n, dtype=int)
    for k in range(n):
        a, b = k % np1, k // np1
        kmap[k] = (p - b) + np1 * a
    for j in range(N):
        for i in range(N):
            e = i + N * j
            e2 = (N - 1 - j) + N * i
            emap[e] = e2
            sig[e2] = prob.sigma[e]
            q[e2][kmap] = prob.q[e]
    fl = np.zeros_like(prob.inflow)
    bmap = np.zeros(fl.shape[0], dtype=int)
    for idx in range(N):
        for node in range(np1):
            # x- (x=0, y=(idx,node)) -> y- (y'=0, x' = 1-y): i' = N-1-idx, a' = p-node
            bmap[bnode_index("x-", idx, node, N, N, p)] = bnode_index("y-", N - 1 - idx, p - node, N, N, p)
            # x+ (x=1) -> y+ (y'=1)
            bmap[bnode_index("x+", idx, node, N, N, p)] = bnode_index("y+", N - 1 - idx, p - node, N, N, p)
            # y- (y=0, x=(idx,node)) -> x+ (x'=1, y'=x): j'=idx, b'=node
            bmap[bnode_index("y-", idx, node, N, N, p)] = bnode_index("x+", idx, node, N, N, p)
            # y+ (y=1) -> x- (x'=0)
            bmap[bnode_index("y+", idx, node, N, N, p)] = bnode_index("x-", idx, node, N, N, p)
    fl[bmap] = prob.inflow
    om = prob.omega.copy()
    om[:, 0], om[:, 1] = -prob.omega[:, 1], prob.omega[:, 0]
    return Problem(prob.name + "-rot", 2, N, N, p, om, prob.w.copy(), sig, q, fl, prob.inv_c_dt), emap, kmap, bmap


@pytest.mark.parametrize("p", [1, 2])
def test_rotation_symmetry(p):
    """90-degree rotation maps phi -> phi, J -> (-Jy, Jx), Txx <-> Tyy, Txy -> -Txy,
    beta and J+ follow their face nodes (SURVEY §8c 'Orientation' pin)."""
    om, w = synth.product_set(4, 16)
    prob = random_problem(21, 2, 4, 4, p, 64, 1, omega=om, w=w)
    rot, emap, kmap, bmap = _rotate90(prob)
    f = oracle.unpack(oracle.sweep(prob), 2, 4, 4, p)
    g = oracle.unpack(oracle.sweep(rot), 2, 4, 4, p)
    sc = np.abs(f["phi"]).max()

    def mapped(a):
        out = np.zeros_like(a)
        for e in range(a.shape[0]):
            out[emap[e]][kmap] = a[e]
        return out

    assert np.abs(g["phi"] - mapped(f["phi"])).max() < 1e-13 * sc
    assert np.abs(g["J"][0] - mapped(-f["J"][1])).max() < 1e-13 * sc
    assert np.abs(g["J"][1] - mapped(f["J"][0])).max() < 1e-13 * sc
    assert np.abs(g["T"][0] - mapped(f["T"][2])).max() < 1e-13 * sc
    assert np.abs(g["T"][2] - mapped(f["T"][0])).max() < 1e-13 * sc
    assert np.abs(g["T"][1] - mapped(-f["T"][1])).max() < 1e-13 * sc
    assert np.abs(g["beta"][bmap] - f["beta"]).max() < 1e-13 * sc
    assert np.abs(g["Jplus"][bmap] - f["Jplus"]).max() < 1e-13 * sc


def test_beta_identity_from_nodal_outputs():
    """R5 reading: beta = 2 J+ - J.n - alpha_n phi at every boundary node, exactly
    (|Omega.n| = 2 max(Omega.n,0) - Omega.n)."""
    prob = random_problem(4, 2, 4, 3, 2, 7, 2)
    f = oracle.unpack(oracle.sweep(prob), 2, 4, 3, 2)
    a = oracle.alpha(prob)
    nx, ny, np1 = 4, 3, 3
    for t in range(f["beta"].size):
        if t < 2 * ny * np1:
            j, b = (t % (ny * np1)) // np1, t % np1
            left = t < ny * np1
            e = (0 if left else nx - 1) + nx * j
            k = (0 if left else 2) + np1 * b
            Jn = -f["J"][0][e, k] if left else f["J"][0][e, k]
            al = a[0] if left else a[1]
        else:
            tt = t - 2 * ny * np1
            i, aa = (tt % (nx * np1)) // np1, tt % np1
            bot = tt < nx * np1
            e = i + nx * (0 if bot else ny - 1)
            k = aa + np1 * (0 if bot else 2)
            Jn = -f["J"][1][e, k] if bot else f["J"][1][e, k]
            al = a[2] if bot else a[3]
        ref = 2 * f["Jplus"][t] - Jn - al * f["phi"][e, k]
        assert abs(f["beta"][t] - ref) < 1e-13 * np.abs(f["phi"]).max()


def test_group_shard_additivity():
    """Gray sums over groups split into shards add up to the full result."""
    prob = random_problem(8, 2, 3, 3, 1, 5, 6)
    full = oracle.sweep(prob)
    parts = oracle.sweep(prob.group_slice(0, 2)) + oracle.sweep(prob.group_slice(2, 6))
    assert np.abs(full - parts).max() < 1e-13 * np.abs(full).max()


def test_configs_generate_small():
    """C1..C5 recipes at reduced size: shapes, positivity, block fraction (R13)."""
    for cfg, kw in ((1, {}), (2, {"nx": 32, "G": 8}), (3, {"nx": 16}), (4, {"nx": 16, "G": 4}), (5, {"nx": 16, "G": 4})):
        P = synth.config(cfg, **kw)
        assert P.sigma.shape == (P.n_el, P.G)
        assert P.q.shape == (P.n_el, P.n, P.G)
        assert P.inflow.shape == (P.n_bnode, P.G)
        assert np.all(P.sigma > 0) and np.all(np.isfinite(P.q))
        assert abs(P.w.sum() - 1.0) < 1e-15
    P = synth.config(3)
    assert np.sum(P.sigma[:, 0] == 2000.0) == 77 * 64


@pytest.mark.parametrize("dim,p", [(1, 2), (2, 1), (2, 2)])
def test_constant_solution_asymmetric_set(dim, p):
    """Constant psi == Q on an ASYMMETRIC random direction set: beta = 0 on every
    face only if alpha is taken per normal as sum w|Omega.n| / sum w (eq:alpha,
    PAPER.md:173-176); phi, J, T, J+ equal their definitions applied to Q."""
    nx, ny = (6, 1) if dim == 1 else (4, 3)
    rng = np.random.default_rng(17)
    ndir = 7
    om, w = synth.configs.random_unit_dirs(rng, ndir, dim)
    if dim == 2:
        om[:, 1] *= 0.3          # make alpha_y clearly differ from alpha_x
        om /= np.linalg.norm(om, axis=1, keepdims=True)
    n = (p + 1) ** dim
    ne = nx * ny
    sig = rng.uniform(0.1, 30.0, size=(ne, 1))
    Q, inv = 2.3, 0.2
    q = np.broadcast_to(((sig + inv) * Q)[:, None, :], (ne, n, 1)).copy()
    nb = 2 if dim == 1 else 2 * (nx + ny) * (p + 1)
    P = Problem("ca", dim, nx, ny, p, om, w, sig, q, np.full((nb, 1), Q), inv)
    f = oracle.unpack(oracle.sweep(P), dim, nx, ny, p)
    assert np.abs(f["phi"] - Q).max() < 1e-13 * Q
    assert np.abs(f["beta"]).max() < 1e-13 * Q
    assert np.abs(f["J"][0] - Q * np.sum(w * om[:, 0])).max() < 1e-13 * Q
    assert np.abs(f["T"][0] - Q * np.sum(w * (om[:, 0] ** 2 - 1 / 3))).max() < 1e-13 * Q
    if dim == 2:
        assert np.abs(f["J"][1] - Q * np.sum(w * om[:, 1])).max() < 1e-13 * Q
        assert np.abs(f["T"][1] - Q * np.sum(w * om[:, 0] * om[:, 1])).max() < 1e-13 * Q
        assert np.abs(f["T"][2] - Q * np.sum(w * (om[:, 1] ** 2 - 1 / 3))).max() < 1e-13 * Q
        t = bnode_index("y+", 1, 0, nx, ny, p)
        assert abs(f["Jplus"][t] - Q * np.sum(w * np.maximum(om[:, 1], 0))) < 1e-13 * Q
    else:
        assert abs(f["Jplus"][1] - Q * np.sum(w * np.maximum(om[:, 0], 0))) < 1e-13 * Q
