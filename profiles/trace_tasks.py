"""Timeline of the persistent 2-D sweep: per task start/end/wait (trace build).
usage: python profiles/trace_tasks.py [cfg] [G_loc]   (G_loc: the first G_loc groups, a group-sharded rank)"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_21784_b200 import build as B  # noqa: E402
import paper_2504_21784_b200.sweep as S  # noqa: E402
import synth  # noqa: E402
import torch  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
so = os.environ.get("TRACE_SO") or "/tmp/libsweep_trace.so"
if not os.environ.get("TRACE_SO"):
    B.build(extra=["-DSWEEP_TRACE"], out=so)
S._lib = None
lib = S.load_library(so)
prob = synth.config(cfg)
if len(sys.argv) > 2:
    prob = prob.group_slice(0, int(sys.argv[2]))
    prob.q, prob.sigma, prob.inflow = (np.ascontiguousarray(x) for x in (prob.q, prob.sigma, prob.inflow))
dev = torch.device("cuda:0")
sig, q, fl = (torch.from_numpy(a).to(dev) for a in (prob.sigma, prob.q, prob.inflow))
sw = S.from_problem(prob)
for _ in range(3):
    sw.sweep_run(sig, prob.inv_c_dt, q, fl)
torch.cuda.synchronize()
st = sw.stats()
sw.timing(True)
sw.sweep_run(sig, prob.inv_c_dt, q, fl)
kt = sw.kernel_times(1)
ntask = 4096
buf = (ctypes.c_longlong * (8 * ntask))()
acc = lib.sweep_debug_trace if prob.p == 2 else lib.sweep_debug_trace_p1  # per-unit trace buffer
acc.argtypes = [ctypes.c_void_p, ctypes.c_int]
acc(buf, ntask)
a = np.array(buf).reshape(-1, 8)
a = a[a[:, 1] > 0]
t0 = a[:, 0].min()
start, end, wait = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2] / 1e3
dur = end - start
print(f"kernel {kt[0, 0]:.3f} ms; tasks {len(a)}; streams {st['streams']}; ctas {st['ctas']}")
print(f"task duration us: mean {dur.mean():.1f} min {dur.min():.1f} max {dur.max():.1f}")
print(f"wait us per task: mean {wait.mean():.1f} max {wait.max():.1f}; total wait fraction {wait.sum() / dur.sum():.3f}")
tot_cyc = dur.sum() * 1e-6 * 1.965e9
print(f"cycles (thread 0): A+wait {a[:, 4].sum() / tot_cyc:.3f}  B {a[:, 5].sum() / tot_cyc:.3f}  rest(C, loop) {1 - (a[:, 4].sum() + a[:, 5].sum()) / tot_cyc:.3f}")
print(f"last end {end.max():.1f} us; sum(dur)/ctas {dur.sum() / st['ctas']:.1f} us")
for k in range(0, len(a), max(1, len(a) // 24)):
    print(f"  task {k:5d} sm {a[k, 3]:3d} start {start[k]:9.1f} end {end[k]:9.1f} wait {wait[k]:8.1f}")
# per-task phase split (thread 0 cycles) of the first tasks (J = 0 strips: no waiting)
for k in range(min(4, len(a))):
    tot = (a[k, 1] - a[k, 0]) * 1e-9 * 1.965e9
    print(f"  task {k}: A+wait {a[k, 4] / tot:.3f}  B {a[k, 5] / tot:.3f}  C+loop {1 - (a[k, 4] + a[k, 5]) / tot:.3f}  "
          f"({(a[k, 1] - a[k, 0]) / 1e3:.1f} us)")
