"""Build libsweep.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsweep.so")
# debug build: device-side bounds checks and trace-ring tags (-DSWEEP_DEBUG), same ABI
DEBUG_LIB = os.path.join(HERE, "libsweep_debug.so")
# device code is split over translation units that compile in parallel
# (k2d_*.cu instantiate the 2-D kernel templates of sweep_device.cuh)
SOURCES = [os.path.join(CSRC, f) for f in ("k2d_p2.cu", "k2d_opt_p2.cu", "k2d_p1.cu", "k2d_opt_p1.cu",
                                           "k_common.cu", "k_1d.cu", "k_trt.cu", "sweep_host.cpp")]
HEADERS = [os.path.join(CSRC, "sweep_internal.h"), os.path.join(CSRC, "sweep_device.cuh"),
           os.path.join(ROOT, "include", "sweep.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2"]
NVCC_FLAGS = [*COMPILE_FLAGS, "-shared", "-ldl"]    # single-command form (experiment builds)


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def compile_objects(out_dir: str, extra=(), verbose: bool = False) -> list:
    """nvcc -c every source in parallel; returns the object paths."""
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(out_dir, exist_ok=True)

    def one(src):
        obj = os.path.join(out_dir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *COMPILE_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        return list(ex.map(one, SOURCES))


def link(objs: list, out: str) -> None:
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", out, *objs, "-ldl"])


def build_debug(force: bool = False) -> str:
    """libsweep_debug.so: the same library with -DSWEEP_DEBUG (tests/test_gpu_debug.py)."""
    if not force and not stale(DEBUG_LIB):
        return DEBUG_LIB
    return build(force=True, extra=("-DSWEEP_DEBUG",), out=DEBUG_LIB)


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    if out == LIB and not extra and not force and not stale():
        return LIB
    tag = f"{os.getpid()}_{abs(hash(tuple(extra))) % 10**8}"
    objs = compile_objects(os.path.join(ROOT, "build", "obj_" + tag), extra, verbose)
    tmp = out + f".tmp{os.getpid()}"
    link(objs, tmp)
    os.replace(tmp, out)
    for o in objs:
        os.remove(o)
    os.rmdir(os.path.dirname(objs[0]))
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
    if "--debug" in sys.argv:
        print(build_debug(force="--force" in sys.argv))
