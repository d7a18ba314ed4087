"""Per-warp wait accounting of the warp-specialised 2-D kernel (trace build).
usage: python profiles/trace_ws.py [cfg]"""
import ctypes, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21784_b200 import build as B  # noqa: E402
import paper_2504_21784_b200.sweep as S  # noqa: E402
import synth  # noqa: E402
import torch  # noqa: E402
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
so = "/tmp/libsweep_trace.so"
subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, "-DSWEEP_TRACE", "-I", os.path.join(ROOT, "include"), "-o", so, *B.SOURCES])
S._lib = None
lib = S.load_library(so)
prob = synth.config(cfg)
dev = torch.device("cuda:0")
sig, q, fl = (torch.from_numpy(a).to(dev) for a in (prob.sigma, prob.q, prob.inflow))
sw = S.from_problem(prob)
for _ in range(2):
    sw.sweep_run(sig, prob.inv_c_dt, q, fl)
torch.cuda.synchronize()
n = 148 * 16
buf = (ctypes.c_longlong * (8 * n))()
lib.sweep_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
zero = (ctypes.c_longlong * (8 * n))()
sw.timing(True)
sw.sweep_run(sig, prob.inv_c_dt, q, fl)
kt = sw.kernel_times(1)
lib.sweep_debug_trace(buf, n)
a = np.array(buf).reshape(148, 16, 8)
cyc = kt[0, 0] * 1e-3 * 1.965e9
comp = a[:, :8, :3].astype(float)
print(f"kernel {kt[0, 0]:.3f} ms = {cyc:.3g} cycles")
print(f"compute warps (fraction of kernel): wait full {comp[:, :, 0].mean() / cyc:.3f}  wait sfree {comp[:, :, 1].mean() / cyc:.3f}  phase B {comp[:, :, 2].mean() / cyc:.3f}")
print(f"X0 predecessor-flag wait (accumulates over 3 runs): {a[:, 8, 3].mean() / cyc / 3:.3f}")
