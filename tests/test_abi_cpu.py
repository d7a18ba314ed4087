"""C-ABI checks that need no GPU (-m "not gpu"): the library builds for sm_100a,
loads, exports every symbol include/sweep.h declares, and its host-side
validation rejects bad descriptions before touching CUDA."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pk():
    from paper_2504_21784_b200 import build
    build.build()
    import paper_2504_21784_b200 as pk
    pk.load_library()
    return pk


def header_functions():
    src = open(os.path.join(ROOT, "include", "sweep.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*\**\s*(\w+)\s*\(", src, flags=re.M)))


def test_header_declares_abi():
    fns = header_functions()
    for f in ("sweep_setup", "sweep_run", "closures_get", "sweep_destroy", "sweep_layout", "sweep_last_error"):
        assert f in fns


def test_library_exports_every_header_symbol(pk):
    lib = pk.load_library()
    for f in header_functions():
        assert hasattr(lib, f), f
    from paper_2504_21784_b200.sweep import EXPORTS
    assert sorted(EXPORTS) == header_functions()


def test_library_is_sm100a(pk):
    so = os.path.join(ROOT, "paper_2504_21784_b200", "libsweep.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _desc(pk, **kw):
    om, w = synth.product_set(2, 8)
    args = dict(dim=2, nx=4, ny=4, p=1, omega=om, w=w, n_group_local=2)
    args.update(kw)
    return args


@pytest.mark.parametrize("bad,code", [
    (dict(dim=3), 1), (dict(p=3), 1), (dict(nx=0), 1), (dict(n_group_local=0), 1), (dict(lx=0.0), 1),
])
def test_setup_rejects_bad_args(pk, bad, code):
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(**_desc(pk, **bad))
    assert ei.value.code == code


def test_setup_rejects_bad_quadrature(pk):
    om, w = synth.product_set(2, 8)
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(**_desc(pk, omega=om, w=w * 1.01))
    assert ei.value.code == pk.sweep.E_QUAD
    om2 = om.copy()
    om2[0] *= 1.001
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(**_desc(pk, omega=om2, w=w))
    assert ei.value.code == pk.sweep.E_QUAD
    w2 = w.copy()
    w2[0], w2[1] = -w2[0], w2[1] + 2 * w2[0]
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(**_desc(pk, omega=om, w=w2))
    assert ei.value.code == pk.sweep.E_QUAD
    omm = np.zeros((4, 3))
    omm[:, 0] = [-1.2, -0.3, 0.3, 0.6]
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(dim=1, nx=4, ny=1, p=1, omega=omm, w=np.full(4, 0.25), n_group_local=1)
    assert ei.value.code == pk.sweep.E_QUAD


def test_setup_without_gpu_fails_loudly(pk):
    """On a box without a CUDA device, a valid description fails with E_CUDA (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pk.SweepError) as ei:
        pk.Sweep(**_desc(pk))
    assert ei.value.code == pk.sweep.E_CUDA


def test_product_never_imports_oracle():
    """The product package and its C sources never reference oracle/."""
    pkg = os.path.join(ROOT, "paper_2504_21784_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "sweep_oracle" not in txt, f
    txt = open(os.path.join(ROOT, "oracle", "sweep_oracle.c")).read()
    includes = re.findall(r'^#include\s*[<"]([^>"]+)[>"]', txt, flags=re.M)
    assert set(includes) <= {"math.h", "stdlib.h", "string.h", "omp.h"}, includes
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            t = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2504_21784_b200" not in t and "from paper_2504_21784_b200" not in t
