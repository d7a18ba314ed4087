"""GPU parity of the NEXT rows (-m gpu) through the C-ABI against the oracle:
  NEXT-1  SWEEP_SIGMA_MOMENTS: sum_g sigma_g phi_g, sum_g sigma_g J_g appended;
  NEXT-2  SWEEP_FIXUP: zero-and-scale negative flux fixup inside the sweep;
  NEXT-3  SWEEP_HALF_RANGE: half-range moments F+, P+ of the consistent method.
Shapes cover both kernels (1-D scan / 2-D strip pipeline), both orders, the
1-group-per-lane and the many-group (16 lanes x 4 groups) layouts, ragged
tails, and problems whose unfixed solution goes negative."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from synth.configs import random_problem
from tests.parity import assert_parity

pytestmark = pytest.mark.gpu

SIG, FIX, HR = oracle.SIGMA_MOMENTS, oracle.FIXUP, oracle.HALF_RANGE


@pytest.fixture(scope="module")
def pk():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device on a -m gpu run")
    from paper_2504_21784_b200 import build
    build.build()
    import paper_2504_21784_b200 as pk
    pk.load_library()
    return pk


def _flags(pk, opts):
    return ((pk.SIGMA_MOMENTS if opts & SIG else 0) | (pk.FIXUP if opts & FIX else 0) |
            (pk.HALF_RANGE if opts & HR else 0))


def check(pk, prob, opts):
    ref = oracle.sweep(prob, opts=opts)
    got = pk.run_problem(prob, flags=_flags(pk, opts))
    return assert_parity(got, ref, prob.dim, prob.nx, prob.ny, prob.p, sigma_moments=bool(opts & SIG),
                         half_range=bool(opts & HR))


def negative_problem(dim, p, nx, ny, G, seed=0, omega=None, w=None):
    """Thick cells and a steep inflow: the unfixed DG solution has negative nodes."""
    prob = random_problem(seed, dim, nx, ny, p, 6 if omega is None else len(w), G, sigma_range=(5.0, 400.0),
                          inv_c_dt=0.1, omega=omega, w=w)
    prob.q[:] = 1e-3
    prob.inflow[:] = 0.0
    prob.inflow[: max(1, prob.inflow.shape[0] // 4)] = 50.0
    return prob


SMALL = [(1, 1, 40, 1, 3), (1, 2, 33, 1, 5), (2, 1, 9, 7, 3), (2, 2, 7, 9, 2), (2, 2, 1, 1, 1), (1, 1, 300, 1, 8)]


@pytest.mark.parametrize("opts", [SIG, FIX, HR, SIG | FIX | HR])
@pytest.mark.parametrize("dim,p,nx,ny,G", SMALL)
def test_options_random_small(pk, opts, dim, p, nx, ny, G):
    prob = random_problem(300 + nx + G, dim, nx, ny, p, 7, G)
    check(pk, prob, opts)


@pytest.mark.parametrize("opts", [FIX, SIG | FIX])
@pytest.mark.parametrize("dim,p,nx,ny", [(1, 2, 12, 1), (2, 1, 6, 5), (2, 2, 6, 5)])  # 1-D p = 1 stays positive
def test_fixup_on_negative_solutions(pk, opts, dim, p, nx, ny):
    prob = negative_problem(dim, p, nx, ny, 3)
    plain = oracle.sweep(prob)
    fixed = oracle.sweep(prob, opts=FIX)
    assert not np.allclose(plain, fixed), "the problem must exercise the fixup"
    check(pk, prob, opts)


@pytest.mark.parametrize("opts", [SIG, FIX, HR | SIG, SIG | FIX | HR])
@pytest.mark.parametrize("nx,ny,G", [(13, 7, 64), (9, 17, 66), (20, 3, 128)])
def test_options_many_group_layout(pk, opts, nx, ny, G):
    om, w = synth.product_set(8, 16)
    if opts & FIX:
        prob = negative_problem(2, 2, nx, ny, G, omega=om, w=w)
    else:
        prob = random_problem(710 + nx, 2, nx, ny, 2, len(w), G, omega=om, w=w)
    check(pk, prob, opts)


@pytest.mark.parametrize("cfg,nx,G", [(4, 24, 5), (5, 24, 64), (2, None, None)])
def test_options_config_recipes(pk, cfg, nx, G):
    prob = synth.config(cfg, nx=nx, G=G) if nx else synth.config(cfg)
    check(pk, prob, SIG | FIX | HR)


def test_half_range_degenerate_directions(pk):
    """Directions with Omega_x = 0 or Omega_y = 0 count in the + half (reading R23), as
    in the sweep's quadrant assignment."""
    om = np.array([[0.0, 0.6, 0.8], [0.6, 0.0, 0.8], [-0.6, 0.0, -0.8], [0.0, -1.0, 0.0], [0.48, -0.6, 0.64]])
    w = np.array([0.1, 0.2, 0.3, 0.25, 0.15])
    prob = random_problem(79, 2, 5, 4, 2, 5, 3, omega=om, w=w)
    check(pk, prob, HR)


def test_fixup_identity_without_negatives(pk):
    """Constant solution: psi == Q > 0, so the fixup never fires."""
    prob = synth.config(5, nx=24, G=64)
    q = np.ascontiguousarray(np.broadcast_to(((prob.sigma + prob.inv_c_dt) * 1.3)[:, None, :], prob.q.shape))
    prob.q = q
    prob.inflow = np.full_like(prob.inflow, 1.3)
    a = pk.run_problem(prob)
    b = pk.run_problem(prob, flags=pk.FIXUP)
    assert np.abs(a - b).max() <= 1e-14 * np.abs(a).max()


def test_sigma_moments_keep_base_fields(pk):
    prob = synth.config(5, nx=24, G=64)
    a = pk.run_problem(prob)
    b = pk.run_problem(prob, flags=pk.SIGMA_MOMENTS)
    assert np.abs(b[:a.size] - a).max() <= 1e-14 * np.abs(a).max()


def test_options_config5_full_size_replicated(pk):
    """C5 at full size (512^2, p = 2, 128 directions, 64 groups: the many-group layout
    and the bench launch configuration) with every option on.  The 64 groups carry the
    data of 4 distinct C5 groups; every output is a sum over groups of per-(d, g) terms
    (the fixup acts per (d, g) too), so gray(GPU) = 16 x sum over the 4 oracle groups."""
    from synth.configs import Problem, replicate_groups
    prob = synth.config(5)
    distinct = [0, 21, 42, 63]
    rep = replicate_groups(prob, distinct)
    opts = SIG | FIX | HR
    got = pk.run_problem(rep, flags=_flags(pk, opts))
    ref = None
    for g in distinct:
        sub = Problem("c5g", 2, 512, 512, 2, prob.omega, prob.w, np.ascontiguousarray(prob.sigma[:, g:g + 1]),
                      np.ascontiguousarray(prob.q[:, :, g:g + 1]), np.ascontiguousarray(prob.inflow[:, g:g + 1]),
                      prob.inv_c_dt)
        r = oracle.sweep(sub, opts=opts)
        ref = r if ref is None else ref + r
    ref *= rep.sigma.shape[1] // len(distinct)
    assert_parity(got, ref, 2, 512, 512, 2, sigma_moments=True, half_range=True)
