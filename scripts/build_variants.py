"""Experiment builds of libsweep.so with -D overrides (plus -DSWEEP_EXPERIMENTS: the SWEEP_CFG /
SWEEP_MAXWARPS layout overrides), into build/<name>.so (bench.py --lib build/<name>.so).
usage: python scripts/build_variants.py name1:-DFOO=1,-DBAR name2: ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21784_b200 import build as b
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
def one(spec):
    name, _, defs = spec.partition(":")
    flags = ["-DSWEEP_EXPERIMENTS"] + [d for d in defs.split(",") if d]
    out = os.path.join(ROOT, "build", name + ".so")
    try:
        b.build(extra=flags, out=out)
        return name, 0, ""
    except subprocess.CalledProcessError as e:
        return name, 1, str(e)
for spec in sys.argv[1:]:   # each build already compiles its units in parallel
    name, rc, err = one(spec)
    print(name, "ok" if rc == 0 else "FAIL\n" + err)
