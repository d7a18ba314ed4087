"""bench.py — DG S_N sweep + fused gray SM closures on B200 (arXiv 2504.21784).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
  (N > 1: launched by torchrun, one rank per GPU, groups sharded, NCCL all-reduce)

One "step" = one full pass of the hot path over the config: sweep of every
(direction, group) with the fused phi/J/T/beta/J+ accumulation, the fixed-order
slab reduction, and (N > 1) the all-reduce of the gray fields.  The default
workload is C5 (BASELINE.json configs[4]); see DESIGN.md §5 for why.

Prints ONE JSON line on rank 0.  `value` = configured unknowns/s (cell-dof x
angle x group, BASELINE.json:2) with inputs resident in HBM; `e2e` = the same
through sweep_run_host with pinned host buffers (H2D of every input and D2H of
the gray output inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DG S_N sweep unknowns/sec (cell-dof×angle×group), % of HBM/FP64 roofline"
SMS, FP64_FMA_PER_SM_CLK, SM_MAX_MHZ = 148, 64, 1965.0
WORKLOAD = {
    1: "C1: 1-D slab, 64 el, p=1, GL S8, 1 group",
    2: "C2: 1-D slab, 1024 el, p=1, GL S16, 64 groups",
    3: "C3: 2-D 128x128, p=1, 4x16 product set (64 dirs), 1 group",
    4: "C4: 2-D 256x256, p=1, 4x16 product set (64 dirs), 32 groups",
    5: "C5: 2-D 512x512, p=2 (9 dofs/el), 8x16 product set (128 dirs), 64 groups",
}


# ------------------------------------------------------------------ algorithmic model
def flops_per_edg(p: int, dim: int, n_dir_quad: int, gb: int) -> float:
    """Flops per (element, distinct direction, group) of the implemented algorithm
    (FMA = 2, reciprocal = 1), counted from the kernel source."""
    if dim == 2 and p == 2:
        # lifts (40 since round 2: the (1,1)/(1,2) pair lifted as half sum and difference,
        # 8 FMA + 4 adds instead of 16 FMA), shifts, reciprocals, scaling, traces
        solve = 40 + 11 + 13 + 33 + 11
        group_sum = 9                             # sum over groups of the 9 modal values
        q_transform = 2 * 81 / n_dir_quad         # modal transform of q per (e, g), per quadrant
        moments = 2 * (6 * 9 + 6 * 81 / n_dir_quad) / gb
        return solve + group_sum + q_transform + moments
    if dim == 2 and p == 1:
        return 8 + 1 + 4 + 1 + 2 + 12 + 20 + 4 + 2 * (6 * 4) / gb
    return 20.0 + 2 * 3 * (p + 1)


def option_flops_per_edg(p: int, dim: int, opts: set) -> float:
    """Extra flops per (element, distinct direction, group) of the NEXT-row options:
    sigma moments: sigma * u accumulated per modal/nodal value (n FMA); fixup, p = 2:
    the nodal check (V (x) V) u, applied axis by axis (58 FMA + 4 adds; the back
    transform of the elements that need the fix is not credited)."""
    n = (p + 1) ** dim
    extra = 0.0
    if "sigma" in opts:
        extra += 2 * n
    if "fixup" in opts and p == 2 and dim == 2:
        extra += 2 * 58 + 4
    return extra


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def profiled_traffic(cfg: int, opts: set):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the sweep kernel from the
    committed ncu --set full capture (profiles/traffic_C<cfg>.json), or None."""
    if opts:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", f"traffic_C{cfg}.json")) as f:
            t = json.load(f)
        return {"bytes_per_launch": t["dram_bytes_per_launch"], "source": t["source"]}
    except Exception:
        return None


def algorithmic_bytes(prob) -> int:
    """Inputs read once + gray output written once."""
    n_in = prob.sigma.size + prob.q.size + prob.inflow.size
    n_out = prob.n_el * prob.n * (1 + prob.dim + (1 if prob.dim == 1 else 3)) + 2 * prob.n_bnode
    return 8 * (n_in + n_out)


def distinct_dirs(prob) -> int:
    if prob.dim == 1:
        return prob.n_dir
    return len({(a, b) for a, b in prob.omega[:, :2].tolist()})


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        try:
            os.unlink(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        loaded = [x for x in sm if x > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


# ------------------------------------------------------------------ distributed plumbing
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def shard_groups(G: int, ws: int, rank: int) -> tuple[int, int]:
    """Contiguous group block of this rank; remainders go to the first ranks."""
    base, rem = divmod(G, ws)
    g0 = rank * base + min(rank, rem)
    return g0, g0 + base + (1 if rank < rem else 0)


# ------------------------------------------------------------------ reference arm: the CPU oracle
def cpu_sample(prob, n_groups: int = 1):
    """Bounded sample of the workload for the CPU oracle: full mesh, every
    direction, the first n_groups groups."""
    return prob.group_slice(0, n_groups)


def run_reference(args, prob) -> dict:
    import oracle
    oracle.build()
    sample = cpu_sample(prob, 1)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.sweep(sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.sweep(sample)
    dt = (time.perf_counter() - t0) / args.steps
    v = sample.unknowns / dt
    desc = f"{prob.name} mesh and all {prob.n_dir} directions, 1 of {prob.G} groups ({sample.unknowns} unknowns)"
    return {"metric": METRIC, "value": v, "unit": "unknowns/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "impl": "reference",
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "sample": desc},
            "cpu_baseline": {"value": v, "unit": "unknowns/s", "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def front_occupancy(prob, n_dir_quad: int, G: int, capacity: int) -> float:
    """sum_k min(active_k, capacity) / (#fronts x capacity) for the anti-diagonal
    fronts k of one quadrant sweep, all quadrants concurrent; a work item is one
    (element, direction, group) solve, capacity = resident lanes x groups per lane."""
    if prob.dim == 1:
        fronts = np.ones(prob.nx)
        nq = 2
    else:
        k = np.arange(prob.nx + prob.ny - 1)
        fronts = np.minimum(np.minimum(k + 1, prob.nx), np.minimum(prob.ny, prob.nx + prob.ny - 1 - k))
        nq = 4
    active = fronts * n_dir_quad * G * nq
    return float(np.minimum(active, capacity).sum() / (fronts.size * capacity))


def graph_replay_ms(sw, run, stream, reps: int = 20):
    """Time of one step replayed from a CUDA graph captured around `run` (the same kernels
    and memsets as the eager step, without the host enqueue cost)."""
    import torch
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        run()   # warm on the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def parity_sample(prob, shard, sw, dev):
    """Oracle-vs-GPU parity on sampled outputs of the bench's own handle (same launch
    configuration as the timed steps, full mesh): every group but the shard's first gets a
    zero source and zero inflow, so the gray output is that one group's contribution; the
    oracle computes group 0 alone.  Returns the per-field errors (tests/parity.py metric)."""
    import torch
    import oracle
    from tests.parity import field_errors, field_ok
    oracle.build()
    q0 = np.zeros_like(shard.q)
    q0[..., 0] = shard.q[..., 0]
    f0 = np.zeros_like(shard.inflow)
    f0[:, 0] = shard.inflow[:, 0]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    sw.sweep_run(t(shard.sigma), prob.inv_c_dt, t(q0), t(f0))
    got = sw.closures_get().cpu().numpy()
    one = shard.group_slice(0, 1)
    t0 = time.perf_counter()
    ref = oracle.sweep(one)
    errs = field_errors(got[:ref.size], ref, prob.dim, prob.nx, prob.ny, prob.p)
    return {"sample": f"group 0 of {shard.G} (others zero), full mesh, all {prob.n_dir} directions, "
                      f"bench launch configuration",
            "max_error": max(e for e, _ in errs.values()),
            "all_pass": all(field_ok(v) for v in errs.values()),
            "fields": {k: [float(e), kind] for k, (e, kind) in errs.items()},
            "oracle_s": time.perf_counter() - t0}


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-floors", action="store_true", help="skip the launch-floor and graph-replay probes "
                                                              "(keeps an ncu launch list to the step's kernels)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--rank-of", type=int, default=1,
                    help="analysis: on one GPU, sweep only the group shard rank 0 of a K-rank group split owns "
                         "(the per-rank workload of the strong-scaling run, without the all-reduce)")
    ap.add_argument("--lib", default=None, help="another build of libsweep.so (experiment builds only, "
                                                  "scripts/build_variants.py)")
    ap.add_argument("--opts", default="", help="comma list of NEXT-row options: sigma (sigma-weighted moments), "
                                                 "fixup (zero-and-scale negative flux fixup), halfrange "
                                                 "(half-range moments of the consistent method), trt (one "
                                                 "outer iteration of the unaccelerated TRT step per step: "
                                                 "emission + sweep + temperature elimination)")
    args = ap.parse_args()
    opts = {o for o in args.opts.split(",") if o}
    if opts - {"sigma", "fixup", "halfrange", "trt"}:
        ap.error(f"unknown --opts {opts - {'sigma', 'fixup', 'halfrange', 'trt'}}")
    if "trt" in opts:
        opts.add("sigma")   # the temperature elimination consumes sum_g sigma_g phi_g
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps

    import synth
    ws, rank, local = dist_env()

    if args.impl == "reference":
        if rank == 0:
            prob = synth.config(args.config)
            print(json.dumps(run_reference(args, prob)), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_2504_21784_b200 as pk

    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if args.lib:
        pk.load_library(args.lib)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)

    prob = synth.config(args.config)
    if args.rank_of > 1 and ws > 1:
        ap.error("--rank-of is a one-process analysis mode")
    g0, g1 = shard_groups(prob.G, max(ws, args.rank_of), rank)
    shard = prob.group_slice(g0, g1)
    job_unknowns = prob.unknowns if args.rank_of == 1 else shard.unknowns
    nid = None
    if ws > 1:
        obj = [pk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    flags = ((pk.SIGMA_MOMENTS if "sigma" in opts else 0) | (pk.FIXUP if "fixup" in opts else 0) |
             (pk.HALF_RANGE if "halfrange" in opts else 0))
    sw = pk.Sweep(prob.dim, prob.nx, prob.ny, prob.p, prob.omega, prob.w, g1 - g0, lx=prob.lx, ly=prob.ly,
                  device=local, fold_z=True, nranks=ws, rank=rank, nccl_id=nid, group_offset=g0,
                  n_group_total=prob.G, flags=flags)
    stream = torch.cuda.current_stream()
    sig = torch.from_numpy(shard.sigma).to(dev)
    q = torch.from_numpy(shard.q).to(dev)
    fl = torch.from_numpy(shard.inflow).to(dev)
    in_bytes = 8 * (sig.numel() + q.numel() + fl.numel())
    l2_bytes = 126 * 2 ** 20
    flush = torch.empty(0, dtype=torch.uint8, device=dev)
    if in_bytes < 2 * l2_bytes:
        # 1 GiB (~0.17 ms of device time per step) also keeps the host's enqueue of the next
        # step (Python + ctypes, tens of microseconds) off the device timeline of tiny configs
        flush = torch.empty(1024 * 2 ** 20, dtype=torch.uint8, device=dev)

    if "trt" in opts:
        # NEXT-4: T^k per element of the config's recipe range, I^k = B_g(T^k) (input generation)
        from synth.planck import group_bounds, planck_groups
        nu = group_bounds(prob.G)[g0:g1 + 1]
        Tk_np = np.repeat(np.random.default_rng(2504).uniform(0.05, 1.0, size=(prob.n_el, 1)), prob.n, axis=1)
        Tk = torch.from_numpy(Tk_np).to(dev)
        Ip = torch.from_numpy(planck_groups(Tk_np, nu).reshape(prob.n_el, prob.n, -1)).to(dev)
        Tout = torch.empty_like(Tk)
        trt_dt = 1.0 / prob.inv_c_dt

    def work():
        if "trt" in opts:
            sw.trt_step(sig, fl, Tk, Ip, nu, cv=1.0, dt=trt_dt, eps=0.0, max_iter=1, T=Tout)
        else:
            sw.sweep_run(sig, prob.inv_c_dt, q, fl)

    def step(evs=None):
        # the L2 flush (small configs) runs before the step's own events
        if flush.numel():
            flush.zero_()
        if evs:
            evs[0].record(stream)
        work()
        if evs:
            evs[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    out = sw.closures_get()  # also surfaces a device error flag before timing

    # ---- timed region
    sw.timing(True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)]
    ev0.record(stream)
    for k in range(args.steps):
        step(step_evs[k])
    ev1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = ev0.elapsed_time(ev1)
    kt = sw.kernel_times(args.steps)
    sw.timing(False)
    # with the flush, a step is timed from its own events (emission, update and the host
    # sync of the TRT option included); without it, over the whole timed region
    step_ms = (float(np.mean([a.elapsed_time(b) for a, b in step_evs])) if flush.numel()
               else total_ms / args.steps)
    t = torch.tensor([step_ms, float(kt[:, 0].mean())], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, sweep_ms = float(t[0]), float(t[1])
    sw.closures_get(out)
    stats = sw.stats()
    launches_per_step = stats["launches"] + (3 if "trt" in opts else 0)  # + emission, update, norm
    # latency floors (C1-C3 are reported against them): an empty kernel launch,
    # and the same step replayed from a CUDA graph
    floors = None
    if "trt" not in opts and not args.no_floors:
        try:
            floors = {"empty_launch_us": pk.launch_floor(local),
                      "graph_replay_ms": graph_replay_ms(sw, lambda: sw.sweep_run(sig, prob.inv_c_dt, q, fl), stream),
                      "launches_per_step": launches_per_step}
            floors["step_floor_ms"] = floors["empty_launch_us"] * launches_per_step * 1e-3
            # the step's device time (graph replay) in units of the empty-launch floor
            floors["graph_replay_over_floor"] = floors["graph_replay_ms"] / floors["step_floor_ms"]
        except Exception as ex:  # noqa: BLE001
            floors = {"error": str(ex)[:200]}

    # ---- end to end through the host API (pinned buffers), same metric
    e2e = None
    if not args.no_e2e and "trt" not in opts:
        hs = torch.from_numpy(shard.sigma).pin_memory()
        hq = torch.from_numpy(shard.q).pin_memory()
        hf = torch.from_numpy(shard.inflow).pin_memory()
        ho = torch.empty(sw.out_size, dtype=torch.float64).pin_memory()
        a_s, a_q, a_f, a_o = hs.numpy(), hq.numpy(), hf.numpy(), ho.numpy()
        sw.sweep_run_host(a_s, prob.inv_c_dt, a_q, a_f, a_o)  # warm (allocates staging)
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            sw.sweep_run_host(a_s, prob.inv_c_dt, a_q, a_f, a_o)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": job_unknowns / (float(te[0]) * 1e-3), "unit": "unknowns/s",
               "ms_per_step": float(te[0]), "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": 8 * sw.out_size,
               "copy": ("pinned H2D in 8-row bands overlapping the sweep (per-band ready flags), then D2H"
                        if prob.dim == 2 else "pinned H2D, sweep, D2H")}

    parity = None
    if ws == 1 and not args.no_parity and not opts:
        parity = parity_sample(prob, shard, sw, dev)

    if rank == 0:
        nd = distinct_dirs(prob)
        gb = min(32, 1 << max(0, (shard.G - 1).bit_length()))
        f_edg = flops_per_edg(prob.p, prob.dim, nd // (4 if prob.dim == 2 else 2), gb) + \
            option_flops_per_edg(prob.p, prob.dim, opts)
        flops = f_edg * prob.n_el * nd * (g1 - g0)             # per rank per launch (folded)
        achieved_tf = flops / (sweep_ms * 1e-3) / 1e12
        peak_nominal = SMS * FP64_FMA_PER_SM_CLK * 2 * SM_MAX_MHZ * 1e6 / 1e12
        peaks = measured_peaks()
        traffic = profiled_traffic(args.config, opts)
        try:
            peak_probe = pk.fp64_probe(local)
        except Exception:
            peak_probe = None
        rec = {
            "metric": METRIC,
            "value": job_unknowns / (step_ms * 1e-3),
            "unit": "unknowns/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config] + (f" + options {sorted(opts)}" if opts else ""),
                       "fold_z": True, "distinct_directions": nd,
                       "unknowns": job_unknowns, "groups_per_rank": g1 - g0,
                       "parallelism": (f"group-sharded x{ws}" + (" + NCCL all-reduce" if ws > 1 else "")) if args.rank_of == 1
                       else f"per-rank workload of a {args.rank_of}-way group split (rank 0, one GPU, no all-reduce)",
                       "l2": ("inputs %.2f GB > 126 MB L2, no flush" % (in_bytes / 1e9)) if not flush.numel()
                       else "1 GiB L2 flush before every step (outside the step's events)"},
            "roofline": {"bound": "alu", "achieved": achieved_tf, "peak": peak_nominal, "unit": "TFLOP/s",
                         "frac": achieved_tf / peak_nominal,
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_source": traffic["source"] if traffic else None,
                         "kernel": "sweep2d_kernel" if prob.dim == 2 else "sweep1d_kernel",
                         "kernel_ms": sweep_ms, "flops_per_launch": flops, "flops_per_edg": f_edg,
                         "peak_source": "FP64 pipe: 148 SM x 64 DFMA/clk x 2 x 1965 MHz (DESIGN.md §5)",
                         "peak_measured_dfma_probe": peak_probe,
                         "frac_of_probe": (achieved_tf / peak_probe) if peak_probe else None,
                         "hbm": {"algorithmic_bytes": algorithmic_bytes(prob),
                                 "achieved_gbs": algorithmic_bytes(prob) / ws / (sweep_ms * 1e-3) / 1e9,
                                 "peak_gbs_measured": peaks.get("hbm_gbs"),
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs (b.copy_(a), read+write)"}},
            "gpu_launches": int(launches_per_step * args.steps),
            "floors": floors,
            "front_occupancy": front_occupancy(prob, nd // (4 if prob.dim == 2 else 2), shard.G,
                                               stats["ctas"] * stats["block"] * stats["groups_per_lane"]),
            "parity": parity,
            "clocks": clk,
            "layout": {k: int(v) for k, v in stats.items()},
            "step_breakdown_ms": {"sweep": float(kt[:, 0].mean()), "finalize": float(kt[:, 1].mean()),
                                  "allreduce": float(kt[:, 2].mean())},
        }
        if e2e:
            rec["e2e"] = e2e
        if not args.no_cpu:
            import oracle
            oracle.build()
            sample = cpu_sample(prob, 1)
            t0 = time.perf_counter()
            oracle.sweep(sample)
            dt = time.perf_counter() - t0
            rec["cpu_baseline"] = {"value": sample.unknowns / dt, "unit": "unknowns/s", "cores": os.cpu_count(),
                                   "kind": "oracle",
                                   "sample": f"{prob.name} mesh, all {prob.n_dir} directions, 1 of {prob.G} groups "
                                             f"({sample.unknowns} unknowns, {dt:.1f} s)"}
            if prob.dim == 1 or prob.n_el * prob.n * prob.n_dir <= 2 ** 25:
                # single-core oracle (C1-C4), same sample
                t0 = time.perf_counter()
                oracle.sweep(sample, nthreads=1)
                d1 = time.perf_counter() - t0
                rec["cpu_baseline"]["single_core"] = {"value": sample.unknowns / d1, "unit": "unknowns/s",
                                                      "cores": 1, "seconds": d1}
        print(json.dumps(rec), flush=True)
    sw.close()
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
