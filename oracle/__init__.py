"""CPU oracle for the DG S_N sweep + gray SM closures (ctypes over sweep_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
paper_2504_21784_b200.  See sweep_oracle.c for what is computed and the
PAPER.md passages each step follows.

Parity status: pinned (tests/test_oracle_pins.py) — dense global assembly in
the paper's jump/average form, closed-form 1-D transmission, constant-solution
exactness, global particle balance, convergence order, rotation symmetry,
quadrature identities; sigma-weighted moments pinned by their reductions
(one group, group-constant sigma, constant solution); the fixup pinned by
the worked element examples and an independent element-by-element sweep in
the jump/average form (tests/dense_dg.py) on tiny meshes; the half-range moments
by an independent psi and isotropic closed forms; the TRT step by the Planck
series, Stefan-Boltzmann, the elimination's fixed point, a brute-force nodal
Newton on the dense global solve, and its outer stop rule (eq:relative_tol) by
rebuilding the iterate sequence from fixed-iteration runs
(tests/test_oracle_next.py::test_trt_stop_rule_rebuilt).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sweep_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile sweep_oracle.c -> liboracle.so (gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        i, d = ctypes.c_int, ctypes.c_double
        lib.oracle_sweep.argtypes = [i, i, i, d, d, i, i, dp, dp, i, dp, d, dp, dp, dp, i]
        lib.oracle_sweep.restype = i
        lib.oracle_sweep2.argtypes = [i, i, i, d, d, i, i, dp, dp, i, dp, d, dp, dp, dp, i, i]
        lib.oracle_sweep2.restype = i
        lib.oracle_out_size2.argtypes = [i, i, i, i, i]
        lib.oracle_out_size2.restype = i
        lib.oracle_fixup.argtypes = [i, dp, dp]
        lib.oracle_fixup.restype = i
        lib.oracle_planck_P.argtypes = [d]
        lib.oracle_planck_P.restype = d
        lib.oracle_planck_groups.argtypes = [d, i, dp, dp]
        lib.oracle_planck_groups.restype = None
        lib.oracle_t_eliminate.argtypes = [d, d, i, dp, dp, d]
        lib.oracle_t_eliminate.restype = d
        lib.oracle_trt_step.argtypes = [i, i, i, d, d, i, i, dp, dp, i, dp, dp, dp, dp, dp, d, d, d, i, dp, dp, i]
        lib.oracle_trt_step.restype = i
        lib.oracle_sweep_psi.argtypes = [i, i, i, d, d, i, i, dp, dp, i, dp, d, dp, dp, i, i, dp, i]
        lib.oracle_sweep_psi.restype = i
        lib.oracle_alpha.argtypes = [i, i, dp, dp, dp]
        lib.oracle_alpha.restype = None
        lib.oracle_out_size.argtypes = [i, i, i, i]
        lib.oracle_out_size.restype = i
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


SIGMA_MOMENTS = 1   # opts bit 0: append sum_g sigma_g phi_g, sum_g sigma_g J_g (NEXT-1)
FIXUP = 2           # opts bit 1: zero-and-scale negative flux fixup inside the sweep (NEXT-2)
HALF_RANGE = 4      # opts bit 2: half-range moments F+, P+ of the consistent method (NEXT-3)


def out_size(dim: int, nx: int, ny: int, p: int, opts: int = 0) -> int:
    return _load().oracle_out_size2(dim, nx, ny if dim == 2 else 1, p, int(opts))


def sweep(prob, nthreads: int = 0, opts: int = 0) -> np.ndarray:
    """Packed gray output phi|J|T|beta|J+ [|sphi|sJ] (same layout as closures_get)."""
    lib = _load()
    om, w, s, q, fl = _c(prob.omega), _c(prob.w), _c(prob.sigma), _c(prob.q), _c(prob.inflow)
    out = np.zeros(out_size(prob.dim, prob.nx, prob.ny, prob.p, opts))
    rc = lib.oracle_sweep2(prob.dim, prob.nx, prob.ny, prob.lx, prob.ly, prob.p, om.shape[0], _ptr(om), _ptr(w),
                           s.shape[1], _ptr(s), float(prob.inv_c_dt), _ptr(q), _ptr(fl), _ptr(out), int(nthreads),
                           int(opts))
    if rc != 0:
        raise RuntimeError(f"oracle_sweep failed rc={rc}")
    return out


def fixup(x, W) -> np.ndarray:
    """The oracle's element-level zero-and-scale fixup applied to a copy of x (weights W)."""
    lib = _load()
    x, W = _c(np.array(x, dtype=np.float64)), _c(W)
    lib.oracle_fixup(x.size, _ptr(W), _ptr(x))
    return x


def planck_P(x: float) -> float:
    """(15/pi^4) int_0^x t^3/(e^t-1) dt by composite Gauss-Legendre quadrature."""
    return _load().oracle_planck_P(float(x))


def planck_groups(T: float, nu) -> np.ndarray:
    """B_g(T) = T^4 [P(nu_{g+1}/T) - P(nu_g/T)] for the bounds nu[0..G] (a = c = 1)."""
    nu = _c(nu)
    out = np.zeros(nu.size - 1)
    _load().oracle_planck_groups(float(T), nu.size - 1, _ptr(nu), _ptr(out))
    return out


def t_eliminate(Tk: float, sphi: float, sigma_g, nu, cv_dt: float) -> float:
    """Root T of cv/dt (T - Tk) + sum_g sigma_g B_g(T) = sphi, by bisection."""
    s, nu = _c(sigma_g), _c(nu)
    return _load().oracle_t_eliminate(float(Tk), float(sphi), s.size, _ptr(s), _ptr(nu), float(cv_dt))


def trt_step(prob, Tk, Iprev, nu, cv: float, dt: float, eps: float = 1e-4, max_iter: int = 50,
             nthreads: int = 0, return_ratios: bool = False):
    """One unaccelerated backward-Euler TRT step (NEXT-4).  prob supplies mesh, quadrature,
    sigma [N_el][G] and inflow; Tk [N_el][n], Iprev [N_el][n][G].  Stops on eq:relative_tol
    (PAPER.md:657-660): ||u^l - u^(l-1)||_2 < eps ||u^1 - u^0||_2 with u = [T, E], E^0 =
    sum_g I^k_g, E^l = phi of the l-th sweep.  Returns (T, iterations) or, with
    return_ratios, (T, iterations, ratios[l-1] = ||u^l - u^(l-1)|| / ||u^1 - u^0||)."""
    lib = _load()
    om, w, s, fl = _c(prob.omega), _c(prob.w), _c(prob.sigma), _c(prob.inflow)
    Tk, Ip, nu = _c(Tk), _c(Iprev), _c(nu)
    T = np.zeros_like(Tk)
    ratios = np.zeros(max(1, int(max_iter)))
    rc = lib.oracle_trt_step(prob.dim, prob.nx, prob.ny, prob.lx, prob.ly, prob.p, om.shape[0], _ptr(om), _ptr(w),
                             s.shape[1], _ptr(s), _ptr(fl), _ptr(Tk), _ptr(Ip), _ptr(nu), float(cv), float(dt),
                             float(eps), int(max_iter), _ptr(T), _ptr(ratios), int(nthreads))
    if rc < 0:
        raise RuntimeError(f"oracle_trt_step failed rc={rc}")
    if return_ratios:
        return T, rc, ratios[:rc].copy()
    return T, rc


def sweep_psi(prob, d: int, g: int, opts: int = 0) -> np.ndarray:
    """psi_{d,g} as [N_el][n]."""
    lib = _load()
    om, w, s, q, fl = _c(prob.omega), _c(prob.w), _c(prob.sigma), _c(prob.q), _c(prob.inflow)
    n = (prob.p + 1) ** prob.dim
    psi = np.zeros((prob.nx * (prob.ny if prob.dim == 2 else 1), n))
    rc = lib.oracle_sweep_psi(prob.dim, prob.nx, prob.ny, prob.lx, prob.ly, prob.p, om.shape[0], _ptr(om), _ptr(w),
                              s.shape[1], _ptr(s), float(prob.inv_c_dt), _ptr(q), _ptr(fl), d, g, _ptr(psi),
                              int(opts))
    if rc != 0:
        raise RuntimeError(f"oracle_sweep_psi failed rc={rc}")
    return psi


def alpha(prob) -> np.ndarray:
    """alpha for outward normals x-, x+, y-, y+ (eq:alpha)."""
    lib = _load()
    om, w = _c(prob.omega), _c(prob.w)
    a = np.zeros(4)
    lib.oracle_alpha(prob.dim, om.shape[0], _ptr(om), _ptr(w), _ptr(a))
    return a


def unpack(out: np.ndarray, dim: int, nx: int, ny: int, p: int, opts: int = 0) -> dict:
    """Split a packed output into named fields (oracle side's own layout reader)."""
    n = (p + 1) ** dim
    nel = nx * (ny if dim == 2 else 1)
    nodes = nel * n
    nb = 2 if dim == 1 else 2 * (nx + ny) * (p + 1)
    o = 0
    f = {}
    f["phi"] = out[o:o + nodes].reshape(nel, n); o += nodes
    f["J"] = out[o:o + dim * nodes].reshape(dim, nel, n); o += dim * nodes
    nT = 1 if dim == 1 else 3
    f["T"] = out[o:o + nT * nodes].reshape(nT, nel, n); o += nT * nodes
    f["beta"] = out[o:o + nb]; o += nb
    f["Jplus"] = out[o:o + nb]; o += nb
    if opts & SIGMA_MOMENTS:
        f["sphi"] = out[o:o + nodes].reshape(nel, n); o += nodes
        f["sJ"] = out[o:o + dim * nodes].reshape(dim, nel, n); o += dim * nodes
    if opts & HALF_RANGE:
        nr = 10 if dim == 2 else 2
        f["HR"] = out[o:o + nr * nodes].reshape(nr, nel, n); o += nr * nodes
    assert o == out.size
    return f
