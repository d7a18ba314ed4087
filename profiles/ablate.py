"""Ablation timing of the 2-D sweep kernel (results are NOT correct for the
ablated variants; timing only).  Builds variants with -D flags into /tmp and
times config C<cfg> through the same C-ABI.  usage: python profiles/ablate.py 5"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21784_b200 import build as B  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
variants = {"base": [], "cfg2_16": [], "cfg2_32": [], "cfg4_16": [], "cfg4_8": [], "nowait": ["-DSWEEP_ABL_NOWAIT"], "nored": ["-DSWEEP_ABL_NORED"],
            "nophaseC": ["-DSWEEP_ABL_NOPHASEC"],
            "all3": ["-DSWEEP_ABL_NOWAIT", "-DSWEEP_ABL_NORED", "-DSWEEP_ABL_NOPHASEC"],
            "nowait_noC": ["-DSWEEP_ABL_NOWAIT", "-DSWEEP_ABL_NOPHASEC"],
            "nowait_nored": ["-DSWEEP_ABL_NOWAIT", "-DSWEEP_ABL_NORED"],
            "c4": ["-DSWEEP_COLS_K4=4"], "c16": ["-DSWEEP_COLS_K4=16"], "c4_nowait": ["-DSWEEP_COLS_K4=4", "-DSWEEP_ABL_NOWAIT"],
            "noprefetch": ["-DSWEEP_NO_PREFETCH"], "noytr": ["-DSWEEP_ABL_NOYTR"], "noytr_nowait": ["-DSWEEP_ABL_NOYTR", "-DSWEEP_ABL_NOWAIT"],
            "nowait_noC_nored_noytr": ["-DSWEEP_ABL_NOYTR", "-DSWEEP_ABL_NOWAIT", "-DSWEEP_ABL_NOPHASEC", "-DSWEEP_ABL_NORED"]}
if len(sys.argv) > 2:
    variants = {k: v for k, v in variants.items() if k in sys.argv[2].split(",")}
import numpy as np  # noqa: E402
import torch  # noqa: E402
import synth  # noqa: E402
import paper_2504_21784_b200.sweep as S  # noqa: E402

prob = synth.config(cfg)
dev = torch.device("cuda:0")
sig = torch.from_numpy(prob.sigma).to(dev)
q = torch.from_numpy(prob.q).to(dev)
fl = torch.from_numpy(prob.inflow).to(dev)
for name, flags in variants.items():
    so = f"/tmp/libsweep_{name}.so"
    cmd = [B.nvcc(), *B.NVCC_FLAGS, *flags, "-I", os.path.join(ROOT, "include"), "-o", so, *B.SOURCES]
    subprocess.check_call(cmd)
    S._lib = None
    S.load_library(so)
    os.environ.pop("SWEEP_CFG", None)
    if name.startswith("cfg"):
        os.environ["SWEEP_CFG"] = name[3:].replace("_", ",")
    sw = S.from_problem(prob)
    for _ in range(3):
        sw.sweep_run(sig, prob.inv_c_dt, q, fl)
    torch.cuda.synchronize()
    sw.timing(True)
    for _ in range(5):
        sw.sweep_run(sig, prob.inv_c_dt, q, fl)
    kt = sw.kernel_times(5)
    print(f"{name:10s} sweep kernel {kt[:, 0].mean():8.3f} ms  (min {kt[:, 0].min():.3f})", flush=True)
    sw.close()
