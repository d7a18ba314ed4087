"""Pins for the oracle's NEXT rows (-m "not gpu"):
  NEXT-1  sigma-weighted gray moments sum_g sigma_g phi_g, sum_g sigma_g J_g
          (eq:sigmaE PAPER.md:183-185, additive MG correction :197-203, :247);
  NEXT-2  zero-and-scale negative flux fixup inside the sweep.
Each pin compares the oracle with something other than itself: an independent
psi (dense global / block assembly in the jump/average form, tests/dense_dg.py),
worked element examples (SPEC.md's fixup examples), or reductions the
definitions fix (one group, group-constant sigma, the constant solution)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from synth.configs import Problem, random_problem
from tests.dense_dg import solve_global, sweep_blocks

SIG, FIX = oracle.SIGMA_MOMENTS, oracle.FIXUP


# ------------------------------------------------------------------ NEXT-1
@pytest.mark.parametrize("dim,p", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_sigma_moments_from_independent_psi(dim, p):
    """sphi = sum_g sigma_g sum_d w psi, sJ = sum_g sigma_g sum_d w Omega psi with psi
    from the dense global solve (not the oracle's sweep)."""
    nx, ny = (5, 1) if dim == 1 else (3, 2)
    prob = random_problem(40 + 3 * dim + p, dim, nx, ny, p, 5, 3)
    f = oracle.unpack(oracle.sweep(prob, opts=SIG), dim, nx, ny, p, opts=SIG)
    sphi = np.zeros_like(f["sphi"])
    sJ = np.zeros_like(f["sJ"])
    for d in range(prob.n_dir):
        for g in range(prob.G):
            psi = solve_global(prob, d, g)
            sg = prob.sigma[:, g][:, None]
            sphi += sg * prob.w[d] * psi
            for c in range(dim):
                sJ[c] += sg * prob.w[d] * prob.omega[d, c] * psi
    scale = np.abs(sphi).max()
    assert np.abs(f["sphi"] - sphi).max() < 1e-13 * scale
    assert np.abs(f["sJ"] - sJ).max() < 1e-13 * scale


@pytest.mark.parametrize("dim,p", [(1, 2), (2, 1)])
def test_sigma_moments_group_constant_sigma(dim, p):
    """sigma_g = s_e for every group => sphi = s_e phi, sJ = s_e J (per element)."""
    nx, ny = (6, 1) if dim == 1 else (4, 3)
    prob = random_problem(61, dim, nx, ny, p, 6, 4)
    s_e = np.exp(np.random.default_rng(3).uniform(-2, 3, size=prob.sigma.shape[0]))
    prob.sigma[:] = s_e[:, None]
    f = oracle.unpack(oracle.sweep(prob, opts=SIG), dim, nx, ny, p, opts=SIG)
    assert np.abs(f["sphi"] - s_e[:, None] * f["phi"]).max() < 1e-13 * np.abs(f["sphi"]).max()
    assert np.abs(f["sJ"] - s_e[None, :, None] * f["J"]).max() < 1e-13 * np.abs(f["sphi"]).max()


def test_sigma_moments_constant_solution():
    """psi == Q_g (constant solution) => sphi = sum_g sigma_g Q_g per node (sigma_t:
    the 1/(c dt) pseudo-absorption is not an opacity), sJ = 0."""
    nx, ny, p, G = 4, 3, 2, 3
    om, w = synth.product_set(4, 8)
    rng = np.random.default_rng(8)
    ne, n = nx * ny, 9
    sig = rng.uniform(0.5, 50.0, size=(ne, G))
    Q = np.array([0.7, 1.9, 0.2])
    inv = 2.5
    q = np.broadcast_to(((sig + inv) * Q)[:, None, :], (ne, n, G)).copy()
    fl = np.broadcast_to(Q, (2 * (nx + ny) * 3, G)).copy()
    prob = Problem("c", 2, nx, ny, p, om, w, sig, q, fl, inv)
    f = oracle.unpack(oracle.sweep(prob, opts=SIG), 2, nx, ny, p, opts=SIG)
    ref = (sig * Q).sum(axis=1)[:, None]
    assert np.abs(f["sphi"] - ref).max() < 1e-13 * ref.max()
    assert np.abs(f["sJ"]).max() < 1e-13 * ref.max()


def test_sigma_moments_leave_base_fields_unchanged():
    prob = random_problem(12, 2, 3, 3, 2, 4, 2)
    a = oracle.sweep(prob)
    b = oracle.sweep(prob, opts=SIG)
    assert np.array_equal(a, b[:a.size])


# ------------------------------------------------------------------ NEXT-2
def test_fixup_worked_examples():
    """SPEC.md fixup examples (1-D p=1, equal weights) and two weighted 2-D cases."""
    W = np.array([0.5, 0.5])
    assert np.array_equal(oracle.fixup([1.0, 2.0], W), [1.0, 2.0])          # unchanged
    assert np.allclose(oracle.fixup([-1.0, 3.0], W), [0.0, 2.0], atol=1e-15)  # average 1 kept
    assert np.array_equal(oracle.fixup([-2.0, 1.0], W), [0.0, 0.0])         # non-positive average
    W4 = np.full(4, 0.25)
    assert np.allclose(oracle.fixup([-1.0, 1.0, 2.0, 2.0], W4), [0.0, 0.8, 1.6, 1.6], atol=1e-15)
    wh = np.array([1.0, 4.0, 1.0]) / 6.0
    W9 = np.outer(wh, wh).reshape(-1)
    x = np.array([1.0, -0.5, 1.0, 2.0, 1.0, 2.0, -0.1, 3.0, 1.0])
    y = oracle.fixup(x, W9)
    assert (y >= 0).all() and y[1] == 0 and y[6] == 0
    assert abs(W9 @ y - W9 @ x) < 1e-15 * abs(W9 @ x)
    assert np.allclose(y[x > 0] / x[x > 0], (W9 @ x) / (W9 @ np.maximum(x, 0)), rtol=1e-15)


def _negative_problem(dim, p, seed):
    """Thick cells, a grazing direction set and steep inflow: the unfixed DG solution
    goes negative somewhere (checked by the tests that use it)."""
    nx, ny = (6, 1) if dim == 1 else (4, 4)
    prob = random_problem(seed, dim, nx, ny, p, 6, 2, sigma_range=(5.0, 400.0), inv_c_dt=0.1)
    prob.q[:] = 1e-3
    prob.inflow[:] = 0.0
    prob.inflow[: max(1, prob.inflow.shape[0] // 4)] = 50.0
    return prob


@pytest.mark.parametrize("dim,p", [(1, 2), (2, 1), (2, 2)])
def test_fixup_sweep_equals_block_substitution(dim, p):
    """psi with the fixup = element-by-element block substitution of the independently
    assembled global system with the fixup applied per element (tests/dense_dg.py)."""
    prob = _negative_problem(dim, p, 0)
    neg = False
    for d in range(prob.n_dir):
        for g in range(prob.G):
            plain = oracle.sweep_psi(prob, d, g)
            neg |= bool((plain < -1e-12 * np.abs(plain).max()).any())
            got = oracle.sweep_psi(prob, d, g, opts=FIX)
            ref = sweep_blocks(prob, d, g, fixup=True)
            assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (d, g)
            assert (got >= 0).all()
    assert neg, "the test problem must exercise the fixup"


def test_fixup_is_identity_without_negatives():
    """Constant solution (psi == Q > 0 everywhere): fixup on and off agree bit for bit."""
    nx, ny, p, G = 4, 3, 2, 2
    om, w = synth.product_set(2, 8)
    sig = np.full((nx * ny, G), 3.0)
    Q = np.array([1.0, 2.0])
    q = np.broadcast_to(((sig + 1.0) * Q)[:, None, :], (nx * ny, 9, G)).copy()
    fl = np.broadcast_to(Q, (2 * (nx + ny) * 3, G)).copy()
    prob = Problem("c", 2, nx, ny, p, om, w, sig, q, fl, 1.0)
    assert np.array_equal(oracle.sweep(prob), oracle.sweep(prob, opts=FIX))


# ------------------------------------------------------------------ NEXT-3
HR = oracle.HALF_RANGE


@pytest.mark.parametrize("dim,p", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_half_range_from_independent_psi(dim, p):
    """F+, P+  = half-range sums of psi from the dense global solve."""
    nx, ny = (5, 1) if dim == 1 else (3, 2)
    prob = random_problem(80 + 3 * dim + p, dim, nx, ny, p, 7, 2)
    f = oracle.unpack(oracle.sweep(prob, opts=HR), dim, nx, ny, p, opts=HR)
    ref = np.zeros_like(f["HR"])
    for d in range(prob.n_dir):
        ox = prob.omega[d, 0]
        oy = prob.omega[d, 1] if dim == 2 else 0.0
        w = prob.w[d]
        rows = [w * ox, w * ox * ox] if dim == 1 else [w * ox, w * oy, w * ox * ox, w * ox * oy, w * oy * oy]
        for g in range(prob.G):
            psi = solve_global(prob, d, g)
            if ox >= 0:
                for m, c in enumerate(rows):
                    ref[m] += c * psi
            if dim == 2 and oy >= 0:
                for m, c in enumerate(rows):
                    ref[5 + m] += c * psi
    assert np.abs(f["HR"] - ref).max() < 1e-13 * np.abs(f["phi"]).max()


def test_half_range_isotropic():
    """psi == Q (constant solution) on a symmetric set: F+_{+x} = Q (alpha_x / 2, 0),
    P+_{+x} = Q (1/6, 0, 1/6 Oy^2 part), likewise for +y — from sum w Omega Omega = I/3
    split evenly by the mirror symmetry, and alpha_n = sum w |Omega.n| (eq:alpha)."""
    nx, ny, p, G = 3, 3, 1, 1
    om, w = synth.product_set(4, 8)
    sig = np.full((nx * ny, G), 2.0)
    q = np.full((nx * ny, 4, G), 3.0)        # sigma~ Q with Q = 1, 1/(c dt) = 1
    fl = np.ones((2 * (nx + ny) * 2, G))
    prob = Problem("iso", 2, nx, ny, p, om, w, sig, q, fl, 1.0)
    f = oracle.unpack(oracle.sweep(prob, opts=HR), 2, nx, ny, p, opts=HR)
    a = oracle.alpha(prob)
    Pyy_half = 0.5 * np.sum(w * om[:, 1] ** 2)
    exp = [a[1] / 2, 0.0, 1 / 6, 0.0, Pyy_half, 0.0, a[3] / 2, np.sum(w * om[:, 0] ** 2) / 2, 0.0, 1 / 6]
    for m, e in enumerate(exp):
        assert np.abs(f["HR"][m] - e).max() < 1e-13, (m, f["HR"][m].ravel()[:3], e)


# ------------------------------------------------------------------ NEXT-4
def _bern_series_P(x):
    """(15/pi^4) int_0^x t^3/(e^t-1) dt by the Bernoulli series (|x| < 2 pi) — a second
    formula for the quadrature the oracle uses."""
    import math
    B = {0: 1.0, 1: -0.5, 2: 1 / 6, 4: -1 / 30, 6: 1 / 42, 8: -1 / 30, 10: 5 / 66, 12: -691 / 2730, 14: 7 / 6,
         16: -3617 / 510, 18: 43867 / 798, 20: -174611 / 330, 22: 854513 / 138, 24: -236364091 / 2730}
    s = sum(b * x ** (k + 3) / (math.factorial(k) * (k + 3)) for k, b in B.items())
    return s * 15 / math.pi ** 4


def test_planck_integral_pins():
    """P(inf) = 1 (int_0^inf t^3/(e^t-1) = pi^4/15); small-x limit; Bernoulli series."""
    import math
    assert abs(oracle.planck_P(1e4) - 1.0) < 1e-15
    x = 1e-3
    assert abs(oracle.planck_P(x) / (15 / math.pi ** 4 * x ** 3 / 3) - 1.0) < 1e-3
    for x in (0.05, 0.5, 1.0, 1.5):
        assert abs(oracle.planck_P(x) - _bern_series_P(x)) < 2e-15, x
    # large x: 1 - (15/pi^4) sum_n e^{-n x} (x^3/n + 3x^2/n^2 + 6x/n^3 + 6/n^4)
    for x in (2.0, 3.0, 5.0, 12.0, 40.0):
        tail = sum(math.exp(-n * x) * (x ** 3 / n + 3 * x ** 2 / n ** 2 + 6 * x / n ** 3 + 6 / n ** 4)
                   for n in range(1, 60))
        assert abs(oracle.planck_P(x) - (1 - 15 / math.pi ** 4 * tail)) < 2e-15, x


def test_stefan_boltzmann():
    """sum_g B_g(T) over bounds covering (0, inf) = T^4 (a = c = 1)."""
    nu = np.concatenate([[0.0], np.logspace(-3, 4, 40)])
    for T in (0.05, 1.0, 7.0):
        assert abs(oracle.planck_groups(T, nu).sum() / T ** 4 - 1.0) < 1e-13


def test_t_elimination_pins():
    """Fixed point (sphi = sum sigma B_g(Tk) => T = Tk), the residual of the root, and
    the heat-capacity-dominated limit T = Tk + (sphi - sum sigma B(Tk)) / (cv/dt + sum sigma B')."""
    nu = synth.planck.group_bounds(6)
    sig = np.array([3.0, 1.0, 0.5, 20.0, 7.0, 0.1])
    Tk = 0.7
    e0 = float(sig @ oracle.planck_groups(Tk, nu))
    assert abs(oracle.t_eliminate(Tk, e0, sig, nu, 5.0) - Tk) < 1e-14
    T = oracle.t_eliminate(Tk, 2.0 * e0, sig, nu, 5.0)
    res = 5.0 * (T - Tk) + sig @ oracle.planck_groups(T, nu) - 2.0 * e0
    assert abs(res) < 1e-13 * 2.0 * e0
    big = 1e5
    T = oracle.t_eliminate(Tk, e0 + 1e-3, sig, nu, big)
    h = 1e-5
    dE = (sig @ oracle.planck_groups(Tk + h, nu) - sig @ oracle.planck_groups(Tk - h, nu)) / (2 * h)
    assert abs((T - Tk) * (big + dE) / 1e-3 - 1.0) < 1e-6   # linearised update


def _trt_problem(dim, p, nx, ny, G, seed=5):
    om, w = synth.slab_set(4) if dim == 1 else synth.product_set(2, 8)
    rng = np.random.default_rng(seed)
    nu = synth.planck.group_bounds(G)
    ne = nx * (ny if dim == 2 else 1)
    n = (p + 1) ** dim
    sig = np.exp(rng.uniform(np.log(0.5), np.log(40.0), size=(ne, G)))
    nb = 2 if dim == 1 else 2 * (nx + ny) * (p + 1)
    Tb = 1.0
    inflow = np.broadcast_to(oracle.planck_groups(Tb, nu), (nb, G)).copy()
    Tk = rng.uniform(0.3, 0.9, size=(ne, n))
    Iprev = np.stack([np.stack([oracle.planck_groups(t, nu) for t in row]) for row in Tk])
    prob = Problem("trt", dim, nx, ny if dim == 2 else 1, p, om, w, sig, np.zeros((ne, n, G)), inflow, 1.0)
    return prob, Tk, Iprev, nu


def test_trt_step_equilibrium():
    """Uniform equilibrium (T = T0 everywhere, I^k = inflow = B_g(T0)) is a fixed point: T
    stays T0.  u^1 - u^0 is rounding noise, so eq:relative_tol (relative to it) either stops
    at once (exactly zero) or runs to max_iter; T = T0 either way."""
    prob, Tk, Iprev, nu = _trt_problem(2, 1, 3, 3, 4)
    T0 = 0.8
    Tk[:] = T0
    Iprev[:] = oracle.planck_groups(T0, nu)
    prob.inflow[:] = oracle.planck_groups(T0, nu)
    T, it = oracle.trt_step(prob, Tk, Iprev, nu, cv=0.3, dt=0.05, eps=1e-12, max_iter=5)
    assert np.abs(T - T0).max() < 1e-13 and 1 <= it <= 5


@pytest.mark.parametrize("dim,p,eps", [(1, 1, 1e-4), (2, 1, 1e-4), (2, 2, 1e-3), (1, 2, 3e-2)])
def test_trt_stop_rule_rebuilt(dim, p, eps):
    """Pin of the outer stopping rule (eq:relative_tol, eps = 1e-4 for the
    unaccelerated scheme PAPER.md:669): rebuild the iterate sequence u^l = [T^l, E^l] from
    fixed-iteration runs (T^l = the l-iteration step, E^l = phi of the sweep on the emission
    of T^(l-1), E^0 = sum_g I^k_g), find the first l >= 2 with ||u^l - u^(l-1)||_2 <
    eps ||u^1 - u^0||_2 here, and require the oracle to stop exactly there with T = T^l."""
    nx, ny, G = (6, 1, 3) if dim == 1 else (3, 3, 3)
    prob, Tk, Iprev, nu = _trt_problem(dim, p, nx, ny, G, seed=11)
    cv, dt = 0.1, 0.05
    ne, n = Tk.shape
    u_prev = np.concatenate([Tk.ravel(), Iprev.sum(axis=-1).ravel()])
    T_prev = Tk
    norms, Ts = [], []
    for l in range(1, 60):
        T_l, it_l = oracle.trt_step(prob, Tk, Iprev, nu, cv=cv, dt=dt, eps=0.0, max_iter=l)
        assert it_l == l
        q = np.zeros((ne, n, G))
        for e in range(ne):
            for k in range(n):
                q[e, k] = prob.sigma[e] * oracle.planck_groups(T_prev[e, k], nu) + Iprev[e, k] / dt
        pr = Problem("rb", prob.dim, prob.nx, prob.ny, p, prob.omega, prob.w, prob.sigma, q, prob.inflow, 1.0 / dt)
        E_l = oracle.sweep(pr)[:ne * n]
        u_l = np.concatenate([T_l.ravel(), E_l])
        norms.append(np.linalg.norm(u_l - u_prev))
        Ts.append(T_l)
        u_prev, T_prev = u_l, T_l
        if l >= 2 and norms[-1] < eps * norms[0]:
            break
    else:
        pytest.fail("sequence did not meet the tolerance in 59 iterations")
    want = len(norms)
    assert want >= 3   # the case exercises more than the first comparison
    T, it, ratios = oracle.trt_step(prob, Tk, Iprev, nu, cv=cv, dt=dt, eps=eps, max_iter=100, return_ratios=True)
    assert it == want
    assert np.array_equal(T, Ts[-1])
    np.testing.assert_allclose(ratios, np.array(norms) / norms[0], rtol=1e-12, atol=0)
    # a tolerance just above the second-to-last ratio stops one iteration earlier (if that
    # is still an iteration >= 2), just below it does not
    if want >= 4:
        _, it_hi = oracle.trt_step(prob, Tk, Iprev, nu, cv=cv, dt=dt, eps=ratios[-2] * (1 + 1e-9), max_iter=100)
        _, it_lo = oracle.trt_step(prob, Tk, Iprev, nu, cv=cv, dt=dt, eps=ratios[-2] * (1 - 1e-9), max_iter=100)
        assert it_hi == want - 1 and it_lo == want


@pytest.mark.parametrize("dim,p", [(1, 1), (2, 1)])
def test_trt_step_fixed_point_brute_force(dim, p):
    """The converged step is the fixed point T = elim(sweep(q(T))); an independent solve:
    Newton on the full nodal vector with psi from the dense global DG solve
    (tests/dense_dg.py) and a finite-difference Jacobian."""
    nx, ny, G = (3, 1, 3) if dim == 1 else (2, 2, 2)
    prob, Tk, Iprev, nu = _trt_problem(dim, p, nx, ny, G)
    cv, dt = 0.4, 0.02
    T_or, it = oracle.trt_step(prob, Tk, Iprev, nu, cv=cv, dt=dt, eps=1e-14, max_iter=200)
    assert it < 200
    ne, n = Tk.shape

    def residual(Tv):
        Tn = Tv.reshape(ne, n)
        q = np.zeros((ne, n, G))
        for e in range(ne):
            for k in range(n):
                q[e, k] = prob.sigma[e] * oracle.planck_groups(Tn[e, k], nu) + Iprev[e, k] / dt
        pr = Problem("fp", prob.dim, prob.nx, prob.ny, p, prob.omega, prob.w, prob.sigma, q, prob.inflow, 1.0 / dt)
        phi = np.zeros((ne, n, G))
        for d in range(pr.n_dir):
            for g in range(G):
                phi[:, :, g] += pr.w[d] * solve_global(pr, d, g)
        r = np.zeros((ne, n))
        for e in range(ne):
            for k in range(n):
                r[e, k] = (cv / dt * (Tn[e, k] - Tk[e, k]) + prob.sigma[e] @ oracle.planck_groups(Tn[e, k], nu)
                           - prob.sigma[e] @ phi[e, k])
        return r.ravel()

    Tv = Tk.ravel().copy()
    for _ in range(30):
        r = residual(Tv)
        Jm = np.zeros((Tv.size, Tv.size))
        for i in range(Tv.size):
            h = 1e-7 * Tv[i]
            Tp = Tv.copy()
            Tp[i] += h
            Jm[:, i] = (residual(Tp) - r) / h
        step = np.linalg.solve(Jm, -r)
        Tv += step
        if np.abs(step).max() < 1e-15 * Tv.max():
            break
    assert np.abs(T_or.ravel() - Tv).max() < 1e-12 * Tv.max()
