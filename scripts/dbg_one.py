"""One random 2-D problem through the C-ABI vs the oracle.
usage: python scripts/dbg_one.py nx ny p n_dir G [build/<name>.so]   (SEED= from the environment)"""
import os
import sys
sys.path.insert(0, '.')
import oracle
from synth.configs import random_problem
import paper_2504_21784_b200 as pk
from tests.parity import field_errors
nx, ny, p, nd, G = map(int, sys.argv[1:6])
lib = sys.argv[6] if len(sys.argv) > 6 else None
if lib:
    pk.load_library(lib)
prob = random_problem(int(os.environ.get("SEED", 507)), 2, nx, ny, p, nd, G)
try:
    got = pk.run_problem(prob)
    ref = oracle.sweep(prob)
    e = field_errors(got, ref, 2, nx, ny, p)
    print(lib or "product", (nx, ny, p, nd, G), 'max err %.2e' % max(v[0] for v in e.values()), flush=True)
except Exception as ex:  # noqa: BLE001
    print(lib or "product", (nx, ny, p, nd, G), 'EXC', ex, flush=True)
