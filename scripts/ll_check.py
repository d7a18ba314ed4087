"""LL ring protocol checks on one GPU: repeated eager runs, CUDA-graph replays and host-API runs of
one handle give bitwise-identical gray outputs and no device error (usage: python scripts/ll_check.py cfg [G])."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_2504_21784_b200.sweep as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = synth.config(cfg)
if len(sys.argv) > 2:
    prob = prob.group_slice(0, int(sys.argv[2]))
    prob.q, prob.sigma, prob.inflow = (np.ascontiguousarray(x) for x in (prob.q, prob.sigma, prob.inflow))
dev = torch.device("cuda:0")
sig, q, fl = (torch.from_numpy(a).to(dev) for a in (prob.sigma, prob.q, prob.inflow))
sw = S.from_problem(prob)
sw.sweep_run(sig, prob.inv_c_dt, q, fl)
ref = sw.closures_get().cpu().clone()
bad = 0
for k in range(20):
    sw.sweep_run(sig, prob.inv_c_dt, q, fl)
    o = sw.closures_get().cpu()
    bad += int(not torch.equal(o, ref))
print("eager runs differing:", bad, flush=True)
stream = torch.cuda.current_stream()
side = torch.cuda.Stream()
side.wait_stream(stream)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(side):
    sw.sweep_run(sig, prob.inv_c_dt, q, fl)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=side):
        sw.sweep_run(sig, prob.inv_c_dt, q, fl)
torch.cuda.synchronize()
bad = 0
for k in range(20):
    g.replay()
    torch.cuda.synchronize()
    o = sw.closures_get().cpu()
    bad += int(not torch.equal(o, ref))
print("graph replays differing:", bad, flush=True)
# graph replays with changed inputs: a stale line would carry the previous replay's values
q2 = q * 1.5
q.copy_(q2)
sw2 = S.from_problem(prob)
sw2.sweep_run(sig, prob.inv_c_dt, q, fl)
ref2 = sw2.closures_get().cpu().clone()
g.replay()
torch.cuda.synchronize()
o = sw.closures_get().cpu()
print("graph replay after input change equals fresh handle:", torch.equal(o, ref2), flush=True)
hs, hq, hf = (x.cpu().numpy() for x in (sig, q, fl))
for k in range(3):
    out = sw.sweep_run_host(hs, prob.inv_c_dt, np.ascontiguousarray(hq), hf)
print("host runs equal:", np.array_equal(out, ref2.numpy()), flush=True)
