"""Seeded synthetic inputs for configs C1..C5 (BASELINE.json:7-11) and random
small problems.  INPUT GENERATION ONLY: no sweep, no closure arithmetic.

Every array is float64, laid out exactly as the C-ABI expects
(include/sweep.h):
  sigma  [N_el][G]        element-constant total opacity sigma_t,g
  q      [N_el][n][G]     nodal isotropic source (reading R2), n = (p+1)^dim
  inflow [N_bnode][G]     isotropic inflow per boundary face node
  omega  [n_dir][3], w [n_dir]   direction set, sum w = 1
Element e = i + nx*j, node k = a + (p+1)*b; boundary face-node order
x- (j, b), x+ (j, b), y- (i, a), y+ (i, a); 1-D: [x=0, x=1].

Seeds: numpy SeedSequence([2504, 21784, cfg, field]).
The readings R7-R14 used for unstated details are listed in DESIGN.md §3.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .planck import group_bounds, group_energy, planck_groups
from .quadrature import product_set, slab_set

F_SIGMA, F_SOURCE, F_BLOCKS, F_NOISE, F_TEMP = 0, 1, 2, 3, 4


def rng_for(cfg: int, fld: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([2504, 21784, cfg, fld])))


@dataclass
class Problem:
    name: str
    dim: int
    nx: int
    ny: int
    p: int
    omega: np.ndarray
    w: np.ndarray
    sigma: np.ndarray
    q: np.ndarray
    inflow: np.ndarray
    inv_c_dt: float
    lx: float = 1.0
    ly: float = 1.0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return (self.p + 1) ** self.dim

    @property
    def n_el(self) -> int:
        return self.nx * self.ny

    @property
    def n_dir(self) -> int:
        return self.omega.shape[0]

    @property
    def G(self) -> int:
        return self.sigma.shape[1]

    @property
    def n_bnode(self) -> int:
        return n_bnode(self.dim, self.nx, self.ny, self.p)

    @property
    def unknowns(self) -> int:
        """cell-dof x angle x group (BASELINE.json:2 metric unit)."""
        return self.n_el * self.n * self.n_dir * self.G

    def group_slice(self, g0: int, g1: int) -> "Problem":
        """The shard a rank owns: groups [g0, g1)."""
        return replace(self, sigma=np.ascontiguousarray(self.sigma[:, g0:g1]),
                       q=np.ascontiguousarray(self.q[:, :, g0:g1]),
                       inflow=np.ascontiguousarray(self.inflow[:, g0:g1]),
                       name=f"{self.name}[g{g0}:{g1}]")


def n_bnode(dim: int, nx: int, ny: int, p: int) -> int:
    if dim == 1:
        return 2
    return 2 * (nx + ny) * (p + 1)


def bnode_index(face: str, idx: int, node: int, nx: int, ny: int, p: int) -> int:
    """Index of boundary face-node (face in x-,x+,y-,y+; idx = j or i; node = b or a)."""
    np1 = p + 1
    if face == "x-":
        return idx * np1 + node
    if face == "x+":
        return ny * np1 + idx * np1 + node
    if face == "y-":
        return 2 * ny * np1 + idx * np1 + node
    if face == "y+":
        return 2 * ny * np1 + nx * np1 + idx * np1 + node
    raise ValueError(face)


def _left_edge_inflow(dim: int, nx: int, ny: int, p: int, values_g: np.ndarray) -> np.ndarray:
    G = values_g.shape[-1]
    inflow = np.zeros((n_bnode(dim, nx, ny, p), G))
    if dim == 1:
        inflow[0, :] = values_g
    else:
        inflow[: ny * (p + 1), :] = values_g[None, :]
    return inflow


def _opaque_blocks(cfg: int, nx: int, ny: int, block: int = 8, frac: float = 0.3) -> np.ndarray:
    """Reading R13: exactly round(frac * N_blocks) 8x8 blocks by seeded permutation.
    Returns a bool mask [ny][nx] (True = opaque)."""
    nbx, nby = -(-nx // block), -(-ny // block)
    nb = nbx * nby
    k = int(round(frac * nb))
    perm = rng_for(cfg, F_BLOCKS).permutation(nb)[:k]
    mask_b = np.zeros(nb, dtype=bool)
    mask_b[perm] = True
    mask_b = mask_b.reshape(nby, nbx)
    mask = np.repeat(np.repeat(mask_b, block, axis=0), block, axis=1)[:ny, :nx]
    return mask


def config(cfg: int, nx: int | None = None, G: int | None = None) -> Problem:
    """Config C<cfg> (1..5) of BASELINE.json; nx / G may be overridden to make
    smaller problems with the same recipe (tests)."""
    if cfg == 1:
        nx = nx or 64
        om, w = slab_set(8)
        sig = rng_for(1, F_SIGMA).uniform(1.0, 10.0, size=(nx, 1))
        q = rng_for(1, F_SOURCE).lognormal(0.0, 1.0, size=(nx, 2, 1))
        inflow = _left_edge_inflow(1, nx, 1, 1, np.ones(1))
        return Problem("C1", 1, nx, 1, 1, om, w, sig, q, inflow, 0.1)
    if cfg == 2:
        nx = nx or 1024
        G = G or 64
        om, w = slab_set(16)
        bnd = group_bounds(G)
        Eg = group_energy(bnd)
        kappa = rng_for(2, F_SIGMA).uniform(0.5, 2.0, size=nx)
        sig = np.clip(kappa[:, None] * Eg[None, :] ** -3, 1e-2, 1e4)
        # nodes of element i at x = i h, (i+1) h  (reading R12: multiplicative noise per node)
        h = 1.0 / nx
        xn = np.stack([np.arange(nx) * h, (np.arange(nx) + 1) * h], axis=1)
        xi = rng_for(2, F_NOISE).uniform(-1.0, 1.0, size=(nx, 2))
        T = (1.0 - 0.9 * xn) * (1.0 + 0.05 * xi)
        B = planck_groups(T, bnd)  # [nx][2][G]
        inv = 0.1
        q = (sig[:, None, :] + inv) * B
        inflow = _left_edge_inflow(1, nx, 1, 1, planck_groups(np.array([1.0]), bnd)[0])
        return Problem("C2", 1, nx, 1, 1, om, w, sig, q, inflow, inv, meta={"bounds": bnd})
    if cfg == 3:
        nx = nx or 128
        om, w = product_set(4, 16)
        mask = _opaque_blocks(3, nx, nx)
        sig = np.where(mask, 2000.0, 0.2).reshape(-1, 1).astype(np.float64)
        q = rng_for(3, F_SOURCE).lognormal(0.0, 1.0, size=(nx * nx, 4, 1))
        inflow = _left_edge_inflow(2, nx, nx, 1, np.ones(1))
        return Problem("C3", 2, nx, nx, 1, om, w, sig, q, inflow, 1.0)
    if cfg in (4, 5):
        if cfg == 4:
            nx = nx or 256
            G = G or 32
            p, (npol, naz), inv = 1, (4, 16), 1.0
        else:
            nx = nx or 512
            G = G or 64
            p, (npol, naz), inv = 2, (8, 16), 10.0
        om, w = product_set(npol, naz)
        bnd = group_bounds(G)
        Eg = group_energy(bnd)
        mask = _opaque_blocks(cfg, nx, nx).reshape(-1)
        kap = np.where(mask, 1000.0, 0.1)
        sig = np.clip(kap[:, None] * Eg[None, :] ** -3, 1e-2, 1e4)
        Te = rng_for(cfg, F_TEMP).uniform(0.05, 1.0, size=nx * nx)
        B = planck_groups(Te, bnd)  # [N_el][G]
        qe = (sig + inv) * B        # reading R11: psi_prev = B_g(T_e) -> q = sigma~ B
        n = (p + 1) ** 2
        q = np.ascontiguousarray(np.broadcast_to(qe[:, None, :], (nx * nx, n, G)))
        inflow = _left_edge_inflow(2, nx, nx, p, planck_groups(np.array([1.0]), bnd)[0])
        return Problem(f"C{cfg}", 2, nx, nx, p, om, w, sig, q, inflow, inv, meta={"bounds": bnd})
    raise ValueError(f"unknown config {cfg}")


def replicate_groups(prob: Problem, distinct: list[int]) -> Problem:
    """Same shapes, but group g carries the data of group distinct[g % len(distinct)].
    The gray result is then (G/len) x the sum over the distinct groups, so an
    oracle of len(distinct) groups checks a full-size run (tests only)."""
    G = prob.G
    src = np.array([distinct[g % len(distinct)] for g in range(G)])
    return replace(prob, sigma=np.ascontiguousarray(prob.sigma[:, src]),
                   q=np.ascontiguousarray(prob.q[:, :, src]),
                   inflow=np.ascontiguousarray(prob.inflow[:, src]),
                   name=prob.name + f"-rep{len(distinct)}")


def random_unit_dirs(rng: np.random.Generator, n_dir: int, dim: int) -> tuple[np.ndarray, np.ndarray]:
    om = np.zeros((n_dir, 3))
    if dim == 1:
        om[:, 0] = rng.uniform(-1.0, 1.0, size=n_dir)
    else:
        v = rng.normal(size=(n_dir, 3))
        om = v / np.linalg.norm(v, axis=1, keepdims=True)
    w = rng.uniform(0.2, 1.0, size=n_dir)
    return om, w / w.sum()


def random_problem(seed: int, dim: int, nx: int, ny: int, p: int, n_dir: int, G: int,
                   sigma_range=(0.05, 50.0), inv_c_dt: float = 0.3, omega=None, w=None) -> Problem:
    """Random small problem: log-uniform sigma, lognormal q, random inflow on every face."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([2504, 21784, 1000, seed])))
    if dim == 1:
        ny = 1
    if omega is None:
        omega, w = random_unit_dirs(rng, n_dir, dim)
    n = (p + 1) ** dim
    ne = nx * ny
    lo, hi = np.log(sigma_range[0]), np.log(sigma_range[1])
    sig = np.exp(rng.uniform(lo, hi, size=(ne, G)))
    q = rng.lognormal(0.0, 1.0, size=(ne, n, G))
    inflow = rng.uniform(0.0, 2.0, size=(n_bnode(dim, nx, ny, p), G))
    return Problem(f"rand{seed}", dim, nx, ny, p, np.ascontiguousarray(omega), np.ascontiguousarray(w),
                   sig, q, inflow, inv_c_dt)
