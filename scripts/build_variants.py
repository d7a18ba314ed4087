"""Experiment builds of libsweep.so with -D overrides, into build/<name>.so (used with SWEEP_LIB=...).
usage: python scripts/build_variants.py name1:-DFOO=1,-DBAR name2: ..."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21784_b200 import build as b
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
def one(spec):
    name, _, defs = spec.partition(":")
    flags = [d for d in defs.split(",") if d]
    out = os.path.join(ROOT, "build", name + ".so")
    cmd = [b.nvcc(), *b.NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"), "-o", out, *b.SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return name, r.returncode, r.stderr[-2000:]
with ThreadPoolExecutor(len(sys.argv) - 1) as ex:
    for name, rc, err in ex.map(one, sys.argv[1:]):
        print(name, "ok" if rc == 0 else "FAIL\n" + err)
