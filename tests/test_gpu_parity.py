"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the CPU oracle on the
same seeded inputs, element by element, relative L-inf <= 1e-11 per field
(north_star), plus full-size property checks in the bench launch configuration."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from synth.configs import Problem, random_problem, replicate_groups
from tests.parity import assert_parity, field_errors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device on a -m gpu run")
    from paper_2504_21784_b200 import build
    build.build()
    import paper_2504_21784_b200 as pk
    pk.load_library()
    return pk


def gpu_out(pk, prob, fold=True):
    return pk.run_problem(prob, fold_z=fold)


def check(pk, prob, fold=True, nthreads=0):
    ref = oracle.sweep(prob, nthreads=nthreads)
    got = gpu_out(pk, prob, fold)
    return assert_parity(got, ref, prob.dim, prob.nx, prob.ny, prob.p)


# ------------------------------------------------------------------ small random
RAND = []
for seed in range(24):
    rng = np.random.default_rng(seed)
    dim = 1 + (seed % 2)
    p = 1 + ((seed // 2) % 2)
    nx = int(rng.integers(1, 10))
    ny = int(rng.integers(1, 10)) if dim == 2 else 1
    G = int(rng.choice([1, 2, 3, 5, 8, 13, 32, 33, 40]))
    nd = int(rng.integers(1, 12))
    RAND.append((seed, dim, nx, ny, p, nd, G))


@pytest.mark.parametrize("seed,dim,nx,ny,p,nd,G", RAND)
def test_random_small(lib, seed, dim, nx, ny, p, nd, G):
    prob = random_problem(500 + seed, dim, nx, ny, p, nd, G)
    check(lib, prob)


@pytest.mark.parametrize("dim,p", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_degenerate_shapes(lib, dim, p):
    """1x1 mesh, one direction, one group; a direction with Omega_x = 0 (R15)."""
    prob = random_problem(77, dim, 1, 1, p, 1, 1)
    check(lib, prob)
    if dim == 2:
        om = np.array([[0.0, 0.6, 0.8], [0.6, 0.0, 0.8], [-0.6, 0.0, -0.8], [0.0, -1.0, 0.0]])
        w = np.array([0.1, 0.2, 0.3, 0.4])
        prob = random_problem(78, 2, 3, 4, p, 4, 3, omega=om, w=w)
        check(lib, prob)


@pytest.mark.parametrize("dim,p,nx,ny", [(2, 1, 37, 21), (2, 2, 19, 33), (1, 1, 300, 1), (1, 2, 257, 1)])
def test_ragged_multi_tile(lib, dim, p, nx, ny):
    """Sizes spanning several strips/chunks/segments with ragged tails."""
    om, w = (synth.product_set(2, 8) if dim == 2 else synth.slab_set(6))
    prob = random_problem(91, dim, nx, ny, p, len(w), 7, omega=om, w=w)
    check(lib, prob)


def test_fold_z_equivalence(lib):
    """z-fold on/off give the same result (reading R20), both equal to the oracle."""
    prob = synth.config(4, nx=24, G=5)
    ref = oracle.sweep(prob)
    a = gpu_out(lib, prob, fold=True)
    b = gpu_out(lib, prob, fold=False)
    assert_parity(a, ref, 2, 24, 24, 1)
    assert_parity(b, ref, 2, 24, 24, 1)


# ------------------------------------------------------------------ many-group layout
# G >= 64, p = 2: 16 lanes x 4 groups per direction (the C5 bench layout), bulk copies
# (G even) or per-element async copies (G odd).  Shapes span several strips / chunks / flag groups
# with ragged tails, meshes smaller than one chunk, and partial group blocks.
MANY = [(1, 1, 64, 4), (3, 2, 64, 8), (13, 7, 64, 8), (9, 17, 66, 4), (33, 5, 130, 8), (6, 11, 65, 4), (2, 9, 128, 8)]


@pytest.mark.parametrize("nx,ny,G,npol", MANY)
def test_many_group_layout(lib, nx, ny, G, npol):
    om, w = synth.product_set(npol, 16)
    prob = random_problem(700 + nx * ny + G, 2, nx, ny, 2, len(w), G, omega=om, w=w)
    check(lib, prob)


# ------------------------------------------------------------------ configs
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_config_full(lib, cfg):
    prob = synth.config(cfg)
    check(lib, prob)


def test_config4_full(lib):
    prob = synth.config(4)
    check(lib, prob)


@pytest.mark.parametrize("cfg,nx,G", [(4, 40, 6), (5, 24, 5), (5, 40, 3)])
def test_config_recipe_reduced(lib, cfg, nx, G):
    prob = synth.config(cfg, nx=nx, G=G)
    check(lib, prob)


def test_config5_full_size_replicated_groups(lib):
    """C5 at full size (512^2, p=2, 128 directions, 64 groups) in the bench launch
    configuration; the 64 groups carry the data of 4 distinct C5 groups, so the
    oracle needs only those 4 groups: gray(GPU) = 16 x sum_{4 groups} oracle."""
    prob = synth.config(5)
    distinct = [0, 21, 42, 63]
    rep = replicate_groups(prob, distinct)
    got = gpu_out(lib, rep)
    small = prob.group_slice(0, 1)
    ref = np.zeros_like(got)
    for g in distinct:
        sub = Problem("c5g", 2, 512, 512, 2, prob.omega, prob.w, np.ascontiguousarray(prob.sigma[:, g:g + 1]),
                      np.ascontiguousarray(prob.q[:, :, g:g + 1]), np.ascontiguousarray(prob.inflow[:, g:g + 1]),
                      prob.inv_c_dt)
        ref += oracle.sweep(sub)
    ref *= len(rep.sigma[0]) // len(distinct)
    del small
    assert_parity(got, ref, 2, 512, 512, 2)


def test_config5_full_all_groups(lib):
    """C5 exactly as BASELINE.json states it and bench.py launches it — 512^2, p = 2, 128
    directions, all 64 distinct groups — against the oracle on every output (the oracle sweeps
    the 64 groups on the host's cores: about 2.5 min on 16 cores)."""
    prob = synth.config(5)
    got = gpu_out(lib, prob)
    ref = oracle.sweep(prob)
    errs = assert_parity(got, ref, 2, 512, 512, 2)
    assert max(e for e, _ in errs.values()) <= 1e-11


# ------------------------------------------------------------------ properties at full size
def _constant_problem(prob, Q=1.3):
    q = np.ascontiguousarray(np.broadcast_to(((prob.sigma + prob.inv_c_dt) * Q)[:, None, :], prob.q.shape))
    fl = np.full_like(prob.inflow, Q)
    return Problem(prob.name + "-const", prob.dim, prob.nx, prob.ny, prob.p, prob.omega, prob.w, prob.sigma, q, fl,
                   prob.inv_c_dt)


@pytest.mark.parametrize("cfg", [4, 5])
def test_constant_solution_full_size(lib, cfg):
    """Infinite-medium constant solution (north_star): psi == Q for every (d, g), so
    phi = G Q, J = T = beta = 0 at every node, on the full-size config data."""
    prob = _constant_problem(synth.config(cfg))
    got = gpu_out(lib, prob)
    import tests.parity as tp
    f = tp.fields(got, 2, prob.nx, prob.ny, prob.p)
    Qs = 1.3 * prob.G
    assert np.abs(f["phi"] - Qs).max() <= 1e-12 * Qs
    for k in ("Jx", "Jy", "Txx", "Txy", "Tyy", "beta"):
        assert np.abs(f[k]).max() <= 1e-12 * Qs, k


def test_beta_identity_full_size(lib):
    """R5: beta = 2 J+ - J.n - alpha_n phi at every boundary node (C5 data, bench config)."""
    prob = synth.config(5)
    got = gpu_out(lib, prob)
    import tests.parity as tp
    f = tp.fields(got, 2, 512, 512, 2)
    a = oracle.alpha(prob)
    N, np1, n = 512, 3, 9
    phi = f["phi"].reshape(-1, n)
    Jx, Jy = f["Jx"].reshape(-1, n), f["Jy"].reshape(-1, n)
    worst = 0.0
    for t in range(f["beta"].size):
        fc, rem = divmod(t, N * np1)
        idx, node = divmod(rem, np1)
        if fc < 2:
            i, j, aa, bb = (0 if fc == 0 else N - 1), idx, (0 if fc == 0 else 2), node
            Jn = -Jx[i + N * j, aa + 3 * bb] if fc == 0 else Jx[i + N * j, aa + 3 * bb]
        else:
            i, j, aa, bb = idx, (0 if fc == 2 else N - 1), node, (0 if fc == 2 else 2)
            Jn = -Jy[i + N * j, aa + 3 * bb] if fc == 2 else Jy[i + N * j, aa + 3 * bb]
        ref = 2 * f["Jplus"][t] - Jn - a[fc] * phi[i + N * j, aa + 3 * bb]
        worst = max(worst, abs(f["beta"][t] - ref))
    assert worst <= 1e-12 * np.abs(phi).max()


def test_group_shards_sum_to_full(lib):
    """Group sharding on one GPU: shards run one after another sum to the full run."""
    prob = synth.config(4, nx=32, G=12)
    full = gpu_out(lib, prob)
    parts = sum(gpu_out(lib, prob.group_slice(a, b)) for a, b in ((0, 3), (3, 8), (8, 12)))
    errs = field_errors(parts, full, 2, 32, 32, 1)
    assert all(e[0] <= 1e-13 for e in errs.values()), errs


def test_deterministic_bitwise(lib):
    prob = synth.config(5, nx=40, G=6)
    a = gpu_out(lib, prob)
    b = gpu_out(lib, prob)
    assert np.array_equal(a, b)


# ------------------------------------------------------------------ errors
def test_sigma_error_flag(lib):
    import paper_2504_21784_b200 as pk
    prob = random_problem(5, 2, 4, 4, 1, 4, 2)
    prob.sigma[3, 1] = -5.0  # sigma~ = -5 + 0.3 < 0
    with pytest.raises(pk.SweepError) as ei:
        gpu_out(lib, prob)
    assert ei.value.code == pk.sweep.E_SIGMA
    prob = random_problem(6, 2, 4, 4, 2, 4, 2)
    prob.q[2, 3, 0] = np.nan
    with pytest.raises(pk.SweepError) as ei:
        gpu_out(lib, prob)
    assert ei.value.code == pk.sweep.E_SIGMA


def test_host_api_matches_device_api(lib):
    import paper_2504_21784_b200 as pk
    prob = synth.config(4, nx=20, G=3)
    a = gpu_out(lib, prob)
    with pk.from_problem(prob) as sw:
        b = sw.sweep_run_host(prob.sigma, prob.inv_c_dt, prob.q, prob.inflow)
    assert np.array_equal(a, b)


def test_nccl_allreduce_plumbing_one_rank(lib):
    """The NCCL path (dlopen of the libnccl torch loaded, ncclGetUniqueId, ncclCommInitRank,
    the in-place ncclAllReduce on the sweep's stream, ncclCommDestroy) on a 1-rank
    communicator (flag SWEEP_FORCE_COMM): the output equals the plain run bit for bit."""
    import torch
    prob = synth.config(4, nx=24, G=6)
    plain = gpu_out(lib, prob)
    nid = lib.nccl_unique_id()
    dev = torch.device("cuda:0")
    with lib.from_problem(prob, nranks=1, rank=0, nccl_id=nid, flags=lib.FORCE_COMM) as sw:
        s, q, f = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (prob.sigma, prob.q, prob.inflow))
        sw.timing(True)
        for _ in range(3):
            sw.sweep_run(s, prob.inv_c_dt, q, f)
        got = sw.closures_get().cpu().numpy()
        kt = sw.kernel_times(3)
    assert np.array_equal(got, plain)
    assert (kt[:, 2] >= 0).all()


# Every 2-D lane layout (groups per lane K, lanes per direction LG; chosen from G) on
# narrow meshes with several strips (ny > rows per strip): the pattern of layouts and
# shapes under which one code-generation of the p = 2 one-group-per-lane kernels once
# faulted (profiles/r01_ncu_c5_sweep2d.md).
LAYOUTS = [(p, G, nx, ny) for p in (1, 2) for G in (1, 2, 5, 8, 16, 33, 64) for nx, ny in ((1, 7), (2, 9), (5, 13))]


@pytest.mark.parametrize("p,G,nx,ny", LAYOUTS)
def test_layout_matrix(lib, p, G, nx, ny):
    prob = random_problem(700 + 10 * G + nx, 2, nx, ny, p, 8, G)
    check(lib, prob)
