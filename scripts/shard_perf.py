"""Per-rank workload of the group-sharded C5 run on one GPU (analysis only: one process,
G_loc groups of C5), for every lane layout override given in SWEEP_CFG_LIST (needs an
experiment build: scripts/build_variants.py, selected with SWEEP_SHARD_LIB=build/<name>.so)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2504_21784_b200.sweep as S
if os.environ.get("SWEEP_SHARD_LIB"): S.load_library(os.environ["SWEEP_SHARD_LIB"])
prob = synth.config(5)
dev = torch.device("cuda:0")
for G in [int(x) for x in sys.argv[1].split(",")]:
    sub = prob.group_slice(0, G)
    s, q, f = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (sub.sigma, sub.q, sub.inflow))
    for cfg in sys.argv[2].split(";"):
        if cfg: os.environ["SWEEP_CFG"] = cfg
        else: os.environ.pop("SWEEP_CFG", None)
        for mw in sys.argv[3].split(","):
            os.environ["SWEEP_MAXWARPS"] = mw
            try:
                sw = S.from_problem(sub)
                for _ in range(2): sw.sweep_run(s, sub.inv_c_dt, q, f)
                torch.cuda.synchronize(); sw.timing(True)
                for _ in range(4): sw.sweep_run(s, sub.inv_c_dt, q, f)
                kt = sw.kernel_times(4); st = sw.stats(); sw.close()
                print(f"G_loc={G:3d} cfg={cfg or 'default':6s} maxwarps={mw} sweep {kt[:,0].mean():7.3f} ms  streams {st['streams']} ctas {st['ctas']}  x{64//G} -> {kt[:,0].mean()*G/64:6.3f} ms per 64-group equivalent", flush=True)
            except Exception as e:
                print(G, cfg, mw, "ERR", e)
