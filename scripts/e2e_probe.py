"""Where the end-to-end C5 step goes: H2D of the inputs alone (one copy / the band pattern),
D2H of the output, the device-resident step, and sweep_run_host (overlapped copy)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
import paper_2504_21784_b200 as pk  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
prob = synth.config(cfg)
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
hs, hq, hf = (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (prob.sigma, prob.q, prob.inflow))
ds, dq, df = (t.to(dev) for t in (hs, hq, hf))
sw = pk.from_problem(prob)
ho = torch.empty(sw.out_size, dtype=torch.float64).pin_memory()


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def h2d_one():
    dq.copy_(hq, non_blocking=True)
    ds.copy_(hs, non_blocking=True)


rows = 8 * prob.nx * prob.G


def h2d_bands():
    fq, fs = dq.view(-1), ds.view(-1)
    gq, gs = hq.view(-1), hs.view(-1)
    nb = (prob.ny + 7) // 8
    for b in range(nb):
        fq[b * rows * prob.q.shape[1]:(b + 1) * rows * prob.q.shape[1]].copy_(
            gq[b * rows * prob.q.shape[1]:(b + 1) * rows * prob.q.shape[1]], non_blocking=True)
        fs[b * rows:(b + 1) * rows].copy_(gs[b * rows:(b + 1) * rows], non_blocking=True)


def d2h():
    ho.copy_(sw.closures_get(), non_blocking=True)


def dev_step():
    sw.sweep_run(ds, prob.inv_c_dt, dq, df)


def host_step():
    sw.sweep_run_host(hs.numpy(), prob.inv_c_dt, hq.numpy(), hf.numpy(), ho.numpy())


gb = (hq.numel() + hs.numel()) * 8 / 1e9
for name, fn in [("h2d one copy", h2d_one), ("h2d bands", h2d_bands), ("d2h out", d2h),
                 ("device step", dev_step), ("run_host", host_step)]:
    t = timed(fn)
    extra = f"  {gb / t * 1e3:.1f} GB/s" if name.startswith("h2d") else ""
    print(f"{name:14s} {t:8.3f} ms{extra}", flush=True)
t0 = time.perf_counter()
for _ in range(5):
    host_step()
print(f"run_host wall {1e3 * (time.perf_counter() - t0) / 5:8.3f} ms")
