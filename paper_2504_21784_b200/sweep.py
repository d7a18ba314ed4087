"""Thin ctypes binding of libsweep.so (include/sweep.h).  Argument marshalling
only: every step of the sweep runs in the library's CUDA kernels.  There is no
CPU fallback — if the library or a CUDA device is missing, construction fails.

PyTorch is used for device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsweep.so")

SWEEP_OK, E_ARG, E_QUAD, E_SIGMA, E_CUDA, E_NCCL, E_INTERNAL = range(7)
FOLD_Z = 1
DETERMINISTIC = 2
SIGMA_MOMENTS = 4   # also return sum_g sigma_g phi_g, sum_g sigma_g J_g (NEXT-1)
FIXUP = 8           # zero-and-scale negative flux fixup inside the sweep (NEXT-2)
HALF_RANGE = 16     # also return the half-range moments F+, P+ of the consistent method (NEXT-3)
FORCE_COMM = 32     # nranks = 1 with a nccl_id: still run the (1-rank) NCCL all-reduce (plumbing tests)
_NAMES = {1: "E_ARG", 2: "E_QUAD", 3: "E_SIGMA", 4: "E_CUDA", 5: "E_NCCL", 6: "E_INTERNAL"}

# every symbol include/sweep.h declares
EXPORTS = ("sweep_setup", "sweep_layout", "sweep_run", "closures_get", "sweep_run_host", "trt_step",
           "sweep_stats", "sweep_timing", "sweep_kernel_times", "sweep_fp64_probe",
           "sweep_nccl_unique_id", "sweep_destroy", "sweep_last_error", "sweep_launch_floor",
           "sweep_selfcheck_solves")


class SweepError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class sweep_desc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("nx", ctypes.c_int), ("ny", ctypes.c_int),
                ("lx", ctypes.c_double), ("ly", ctypes.c_double), ("p", ctypes.c_int),
                ("n_dir", ctypes.c_int), ("omega", ctypes.POINTER(ctypes.c_double)),
                ("w", ctypes.POINTER(ctypes.c_double)), ("n_group_local", ctypes.c_int),
                ("group_offset", ctypes.c_int), ("n_group_total", ctypes.c_int), ("device", ctypes.c_int),
                ("nranks", ctypes.c_int), ("rank", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("flags", ctypes.c_uint)]


class trt_params(ctypes.Structure):
    _fields_ = [("nu", ctypes.POINTER(ctypes.c_double)), ("cv", ctypes.c_double), ("dt", ctypes.c_double),
                ("eps", ctypes.c_double), ("max_iter", ctypes.c_int), ("ratios", ctypes.POINTER(ctypes.c_double))]


_lib = None


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load libsweep.so (fails loudly if it has not been built).  `path` selects another
    build of the same library (experiment builds, scripts/build_variants.py); it must be
    given before the first load."""
    global _lib
    if _lib is not None and path is not None and os.path.abspath(path) != _lib._name_abs:
        raise RuntimeError(f"libsweep already loaded from {_lib._name_abs}")
    path = path or LIB_PATH
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run `python -m paper_2504_21784_b200.build` "
                               "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(path)
        vp, sz, dp, i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int
        lib.sweep_setup.argtypes = [ctypes.POINTER(sweep_desc), ctypes.POINTER(vp)]
        lib.sweep_setup.restype = i
        lib.sweep_layout.argtypes = [vp, ctypes.POINTER(sz), ctypes.POINTER(sz)]
        lib.sweep_layout.restype = i
        lib.sweep_run.argtypes = [vp, dp, ctypes.c_double, dp, dp, vp]
        lib.sweep_run.restype = i
        lib.closures_get.argtypes = [vp, dp, sz, vp]
        lib.closures_get.restype = i
        lib.sweep_run_host.argtypes = [vp, dp, ctypes.c_double, dp, dp, dp, sz, vp]
        lib.sweep_run_host.restype = i
        lib.trt_step.argtypes = [vp, dp, dp, dp, dp, ctypes.POINTER(trt_params), dp, ctypes.POINTER(i), vp]
        lib.trt_step.restype = i
        lib.sweep_stats.argtypes = [vp, ctypes.POINTER(ctypes.c_longlong)]
        lib.sweep_stats.restype = i
        lib.sweep_timing.argtypes = [vp, i]
        lib.sweep_timing.restype = i
        lib.sweep_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), i, ctypes.POINTER(i)]
        lib.sweep_kernel_times.restype = i
        lib.sweep_fp64_probe.argtypes = [i, ctypes.POINTER(ctypes.c_double)]
        lib.sweep_fp64_probe.restype = i
        lib.sweep_selfcheck_solves.argtypes = [i, i, i, ctypes.c_ulonglong, ctypes.POINTER(ctypes.c_double)]
        lib.sweep_selfcheck_solves.restype = i
        lib.sweep_launch_floor.argtypes = [i, i, ctypes.POINTER(ctypes.c_double)]
        lib.sweep_launch_floor.restype = i
        lib.sweep_nccl_unique_id.argtypes = [vp]
        lib.sweep_nccl_unique_id.restype = i
        lib.sweep_destroy.argtypes = [vp]
        lib.sweep_destroy.restype = None
        lib.sweep_last_error.argtypes = [vp]
        lib.sweep_last_error.restype = ctypes.c_char_p
        lib._name_abs = os.path.abspath(path)
        _lib = lib
    return _lib


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    rc = lib.sweep_nccl_unique_id(buf)
    if rc:
        raise SweepError(rc, lib.sweep_last_error(None).decode())
    return buf.raw


def fp64_probe(device: int = 0) -> float:
    """Measured FP64 FMA throughput of the device in TFLOP/s."""
    lib = load_library()
    t = ctypes.c_double()
    rc = lib.sweep_fp64_probe(device, ctypes.byref(t))
    if rc:
        raise SweepError(rc, lib.sweep_last_error(None).decode())
    return t.value


def launch_floor(device: int = 0, reps: int = 2000) -> float:
    """Device time per launch of an empty kernel, back to back on one stream (microseconds)."""
    lib = load_library()
    t = ctypes.c_double()
    rc = lib.sweep_launch_floor(device, reps, ctypes.byref(t))
    if rc:
        raise SweepError(rc, lib.sweep_last_error(None).decode())
    return t.value


def selfcheck_solves(p: int, n: int = 1 << 20, seed: int = 1, device: int = 0) -> float:
    """Largest relative difference between the sweep's structured element solves and a plain
    dense LU of the same random element systems, both on the device (include/sweep.h)."""
    lib = load_library()
    r = ctypes.c_double()
    rc = lib.sweep_selfcheck_solves(device, p, n, seed, ctypes.byref(r))
    if rc:
        raise SweepError(rc, lib.sweep_last_error(None).decode())
    return r.value


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _check_dev(name: str, t, numel: int, device: int) -> None:
    """A contiguous float64 CUDA tensor on `device` with exactly `numel` elements."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    if t.device.index != device:
        raise ValueError(f"{name} is on cuda:{t.device.index}, the handle on cuda:{device}")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")


def _check_host(name: str, a, numel: int) -> None:
    """A C-contiguous float64 numpy array with exactly `numel` elements."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"{name} must be a C-contiguous float64 numpy array")
    if a.size != numel:
        raise ValueError(f"{name} has {a.size} elements, expected {numel}")


class Sweep:
    """One sweep configuration (mesh, order, quadrature, group shard) on one GPU."""

    def __init__(self, dim: int, nx: int, ny: int, p: int, omega, w, n_group_local: int,
                 lx: float = 1.0, ly: float = 1.0, device: int = 0, fold_z: bool = True,
                 nranks: int = 1, rank: int = 0, nccl_id: bytes | None = None,
                 group_offset: int = 0, n_group_total: int | None = None, flags: int = 0):
        self._lib = load_library()
        self._om = np.ascontiguousarray(omega, dtype=np.float64).reshape(-1, 3)
        self._w = np.ascontiguousarray(w, dtype=np.float64).reshape(-1)
        d = sweep_desc()
        d.dim, d.nx, d.ny, d.lx, d.ly, d.p = dim, nx, (ny if dim == 2 else 1), lx, ly, p
        d.n_dir = self._om.shape[0]
        d.omega, d.w = _dptr(self._om), _dptr(self._w)
        d.n_group_local = n_group_local
        d.group_offset = group_offset
        d.n_group_total = n_group_total if n_group_total is not None else n_group_local
        d.device, d.nranks, d.rank = device, nranks, rank
        self._id = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        d.nccl_id = ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None
        d.flags = (FOLD_Z if fold_z else 0) | int(flags)
        h = ctypes.c_void_p()
        rc = self._lib.sweep_setup(ctypes.byref(d), ctypes.byref(h))
        if rc:
            raise SweepError(rc, self._lib.sweep_last_error(None).decode())
        self._h = h
        self.dim, self.nx, self.ny, self.p, self.G = dim, nx, (ny if dim == 2 else 1), p, n_group_local
        self.device = device
        off = (ctypes.c_size_t * 8)()
        tot = ctypes.c_size_t()
        self._check(self._lib.sweep_layout(self._h, off, ctypes.byref(tot)))
        self.offsets = list(off)
        self.out_size = tot.value
        self.n = (p + 1) ** dim
        self.n_el = nx * self.ny
        self.n_bnode = 2 if dim == 1 else 2 * (nx + self.ny) * (p + 1)

    # ---------------------------------------------------------------- helpers
    def _check(self, rc: int):
        if rc:
            raise SweepError(rc, self._lib.sweep_last_error(self._h).decode())

    @staticmethod
    def _stream_ptr(stream) -> int | None:
        if stream is None:
            import torch
            return torch.cuda.current_stream().cuda_stream
        return int(stream)

    # ---------------------------------------------------------------- ABI calls
    def sweep_run(self, sigma, inv_c_dt: float, q, inflow, stream=None) -> None:
        """sigma [N_el][G], q [N_el][n][G], inflow [N_bnode][G]: contiguous float64 CUDA tensors."""
        _check_dev("sigma", sigma, self.n_el * self.G, self.device)
        _check_dev("q", q, self.n_el * self.n * self.G, self.device)
        _check_dev("inflow", inflow, self.n_bnode * self.G, self.device)
        self._check(self._lib.sweep_run(self._h, sigma.data_ptr(), float(inv_c_dt), q.data_ptr(),
                                        inflow.data_ptr(), self._stream_ptr(stream)))

    def closures_get(self, out=None, stream=None):
        """Packed gray output phi|J|T|beta|J+ into out (device or host tensor)."""
        import torch
        if out is None:
            out = torch.empty(self.out_size, dtype=torch.float64, device=f"cuda:{self.device}")
        if not isinstance(out, torch.Tensor) or out.dtype != torch.float64 or not out.is_contiguous():
            raise ValueError("out must be a contiguous float64 tensor")
        if out.is_cuda and out.device.index != self.device:
            raise ValueError(f"out is on cuda:{out.device.index}, the handle on cuda:{self.device}")
        self._check(self._lib.closures_get(self._h, out.data_ptr(), out.numel(), self._stream_ptr(stream)))
        return out

    def sweep_run_host(self, sigma: np.ndarray, inv_c_dt: float, q: np.ndarray, inflow: np.ndarray,
                       out: np.ndarray | None = None, stream=None) -> np.ndarray:
        """End-to-end with host arrays (pinned numpy views of torch pinned tensors recommended)."""
        if out is None:
            out = np.empty(self.out_size)
        _check_host("sigma", sigma, self.n_el * self.G)
        _check_host("q", q, self.n_el * self.n * self.G)
        _check_host("inflow", inflow, self.n_bnode * self.G)
        if not isinstance(out, np.ndarray) or out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"] or \
                not out.flags["WRITEABLE"]:
            raise ValueError("out must be a writeable C-contiguous float64 numpy array")
        self._check(self._lib.sweep_run_host(self._h, sigma.ctypes.data, float(inv_c_dt), q.ctypes.data,
                                             inflow.ctypes.data, out.ctypes.data, out.size,
                                             self._stream_ptr(stream)))
        return out

    def trt_step(self, sigma, inflow, Tk, Iprev, nu, cv: float, dt: float, eps: float = 1e-4, max_iter: int = 50,
                 T=None, stream=None, return_ratios: bool = False):
        """One unaccelerated backward-Euler TRT step (include/sweep.h trt_step): CUDA float64
        tensors sigma [N_el][G], inflow [N_bnode][G], Tk [N_el][n], Iprev [N_el][n][G];
        nu: host group bounds [G+1].  Returns (T tensor [N_el][n], outer iterations) or, with
        return_ratios, also ||u^l - u^(l-1)|| / ||u^1 - u^0|| per iteration (eq:relative_tol)."""
        _check_dev("sigma", sigma, self.n_el * self.G, self.device)
        _check_dev("inflow", inflow, self.n_bnode * self.G, self.device)
        _check_dev("Tk", Tk, self.n_el * self.n, self.device)
        _check_dev("Iprev", Iprev, self.n_el * self.n * self.G, self.device)
        if T is None:
            import torch
            T = torch.empty_like(Tk)
        _check_dev("T", T, self.n_el * self.n, self.device)
        if int(max_iter) < 1:
            raise ValueError("max_iter must be >= 1")
        nu_a = np.ascontiguousarray(nu, dtype=np.float64).reshape(-1)
        if nu_a.size != self.G + 1:
            raise ValueError(f"nu has {nu_a.size} bounds, expected G + 1 = {self.G + 1}")
        ratios = np.zeros(int(max_iter))
        prm = trt_params(_dptr(nu_a), float(cv), float(dt), float(eps), int(max_iter), _dptr(ratios))
        it = ctypes.c_int()
        self._check(self._lib.trt_step(self._h, sigma.data_ptr(), inflow.data_ptr(), Tk.data_ptr(), Iprev.data_ptr(),
                                       ctypes.byref(prm), T.data_ptr(), ctypes.byref(it), self._stream_ptr(stream)))
        if return_ratios:
            return T, it.value, ratios[:it.value].copy()
        return T, it.value

    def stats(self) -> dict:
        a = (ctypes.c_longlong * 8)()
        self._check(self._lib.sweep_stats(self._h, a))
        return {"launches": a[0], "directions_swept": a[1], "streams": a[2], "ctas": a[3], "block": a[4],
                "groups_per_lane": a[5], "lanes_per_direction": a[6], "sms": a[7]}

    def timing(self, enable: bool = True) -> None:
        self._check(self._lib.sweep_timing(self._h, 1 if enable else 0))

    def kernel_times(self, max_runs: int = 1024) -> np.ndarray:
        """[runs][3] ms: sweep kernel, finalize kernel, all-reduce."""
        buf = (ctypes.c_double * (3 * max_runs))()
        n = ctypes.c_int()
        self._check(self._lib.sweep_kernel_times(self._h, buf, max_runs, ctypes.byref(n)))
        return np.array(buf[:3 * n.value]).reshape(n.value, 3)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sweep_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def unpack(self, out) -> dict:
        """Named views of a packed output (numpy or torch)."""
        n = (self.p + 1) ** self.dim
        nel = self.nx * self.ny
        o = self.offsets
        nT = 1 if self.dim == 1 else 3
        f = {"phi": out[o[0]:o[1]].reshape(nel, n), "J": out[o[1]:o[2]].reshape(self.dim, nel, n),
             "T": out[o[2]:o[3]].reshape(nT, nel, n), "beta": out[o[3]:o[4]], "Jplus": out[o[4]:o[5]]}
        if o[5] < o[7]:
            f["sphi"] = out[o[5]:o[6]].reshape(nel, n)
            f["sJ"] = out[o[6]:o[7]].reshape(self.dim, nel, n)
        if o[7] < self.out_size:
            f["HR"] = out[o[7]:].reshape(-1, nel, n)
        return f


def from_problem(prob, device: int = 0, fold_z: bool = True, **kw) -> Sweep:
    """Sweep handle for a synth.Problem-like object (dim, nx, ny, p, omega, w, G, lx, ly)."""
    return Sweep(prob.dim, prob.nx, prob.ny, prob.p, prob.omega, prob.w, prob.sigma.shape[1],
                 lx=prob.lx, ly=prob.ly, device=device, fold_z=fold_z, **kw)


def run_problem(prob, device: int = 0, fold_z: bool = True, flags: int = 0) -> np.ndarray:
    """Convenience: copy a problem to the GPU, sweep once, return the packed output (numpy)."""
    import torch
    dev = torch.device(f"cuda:{device}")
    with from_problem(prob, device, fold_z, flags=flags) as sw:
        s = torch.from_numpy(np.ascontiguousarray(prob.sigma)).to(dev)
        q = torch.from_numpy(np.ascontiguousarray(prob.q)).to(dev)
        f = torch.from_numpy(np.ascontiguousarray(prob.inflow)).to(dev)
        sw.sweep_run(s, prob.inv_c_dt, q, f)
        out = sw.closures_get()
        return out.cpu().numpy()
