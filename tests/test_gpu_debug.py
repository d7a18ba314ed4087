"""The debug build (libsweep_debug.so, -DSWEEP_DEBUG) on small shapes (-m gpu): every global
index of the kernels is bounds-checked and every strip-boundary trace read checks that the
ring slot was written by the strip below in this run (a failed check raises E_SIGMA with
"debug check failed" from closures_get).  Runs in a subprocess: one process loads one build
of the library.  The shapes cover every 2-D lane layout (G from 1 to 130), several strips and
chunks with ragged tails, both orders, the 1-D scan, and the options."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys
sys.path.insert(0, ".")
import numpy as np
import oracle, synth
from synth.configs import random_problem
from paper_2504_21784_b200 import build
import paper_2504_21784_b200 as pk
pk.load_library(build.build_debug())
from tests.parity import assert_parity
cases = []
for p in (1, 2):
    for G in (1, 3, 8, 16, 33, 64, 130):
        for nx, ny in ((1, 1), (5, 13), (19, 6)):
            cases.append((2, p, nx, ny, 8 if G < 64 else 16, G, 0))
cases += [(1, 1, 70, 1, 8, 5, 0), (1, 2, 33, 1, 6, 40, 0), (1, 1, 40, 1, 4, 3, 7)]
cases += [(2, 2, 9, 7, 16, 64, 1), (2, 1, 9, 7, 8, 6, 2), (2, 2, 6, 11, 8, 5, 4)]
for i, (dim, p, nx, ny, nd, G, opts) in enumerate(cases):
    prob = random_problem(77_000 + i, dim, nx, ny, p, nd, G)
    flags = ((pk.SIGMA_MOMENTS if opts & 1 else 0) | (pk.FIXUP if opts & 2 else 0) |
             (pk.HALF_RANGE if opts & 4 else 0))
    got = pk.run_problem(prob, flags=flags)
    ref = oracle.sweep(prob, opts=opts)
    assert_parity(got, ref, dim, prob.nx, prob.ny, p, sigma_moments=bool(opts & 1), half_range=bool(opts & 4))
print("debug build ok", len(cases))
'''


def test_debug_build_small_shapes():
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "debug build ok" in r.stdout
