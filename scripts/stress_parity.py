"""Randomised GPU-vs-oracle parity sweep over shapes, orders, lane layouts and options
(evidence beyond the pytest cases).  usage: python scripts/stress_parity.py N seed"""
import os, sys, time
sys.path.insert(0, '.')
import numpy as np
import oracle, synth
from synth.configs import random_problem
import paper_2504_21784_b200 as pk
from tests.parity import field_errors, field_ok

n, seed = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
worst, fails, ran = 0.0, 0, 0
t0 = time.time()
for i in range(n):
    dim = int(rng.integers(1, 3))
    p = int(rng.integers(1, 3))
    nx = int(rng.integers(1, 40 if dim == 2 else 300))
    ny = int(rng.integers(1, 40)) if dim == 2 else 1
    G = int(rng.choice([1, 2, 3, 7, 16, 17, 31, 32, 40, 64, 65, 66, 100, 128]))
    if dim == 2 and rng.random() < 0.5:
        om, w = synth.product_set(int(rng.choice([2, 4, 8])), int(rng.choice([4, 8, 16])))
        nd = len(w)
    else:
        om = w = None
        nd = int(rng.integers(1, 20))
    opts = int(rng.integers(0, 8)) if rng.random() < 0.5 else 0
    if nx * ny * G * nd > 4_000_000:
        continue
    ran += 1
    prob = random_problem(10_000 + seed * 1000 + i, dim, nx, ny, p, nd, G, omega=om, w=w)
    flags = ((pk.SIGMA_MOMENTS if opts & 1 else 0) | (pk.FIXUP if opts & 2 else 0) | (pk.HALF_RANGE if opts & 4 else 0))
    try:
        got = pk.run_problem(prob, flags=flags)
        ref = oracle.sweep(prob, opts=opts)
        e = field_errors(got, ref, dim, nx, ny, p, bool(opts & 1), bool(opts & 4))
        m = max(v[0] for v in e.values())
        worst = max(worst, m)
        ok = all(field_ok(v) for v in e.values())
    except Exception as ex:  # noqa: BLE001
        ok, m = False, float("nan")
        print("EXC", ex)
    if ok and m > 1e-13:
        worst_k = max(e, key=lambda k: e[k][0])
        print(f"note dim={dim} p={p} nx={nx} ny={ny} G={G} nd={nd} opts={opts} err={m:.2e} field={worst_k}", flush=True)
    if not ok:
        fails += 1
        print(f"FAIL i={i} dim={dim} p={p} nx={nx} ny={ny} G={G} nd={nd} opts={opts} err={m:.2e}", flush=True)
        if np.isfinite(m):
            print("     ", {k: (f"{v[0]:.2e}", v[1]) for k, v in e.items()}, flush=True)
            print("      omega", np.round(prob.omega, 4).tolist(), "w", np.round(prob.w, 4).tolist(), flush=True)
print(f"{ran} of {n} cases run, {fails} failures, worst relative error {worst:.2e}, {time.time() - t0:.0f} s", flush=True)
