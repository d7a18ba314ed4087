"""bench.py contract checks that run on CPU (-m "not gpu"): the reference arm (the CPU
oracle, bench.py --impl reference) prints one JSON line with the keys the driver reads,
and the algorithmic model used for the roofline is internally consistent."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["unit"] == d["unit"]
    assert d["config"]["workload"].startswith("C1")


def test_roofline_model():
    sys.path.insert(0, ROOT)
    import bench
    import synth
    # C5: 132.4 flops per (element, distinct direction, group) with 16 directions per quadrant
    # (144.4 before the round-2 half-sum / half-difference lifts: 40 instead of 52 lift flops)
    f = bench.flops_per_edg(2, 2, 16, 32)
    assert 130 < f < 135
    prob = synth.config(1)
    assert bench.algorithmic_bytes(prob) == 8 * (prob.sigma.size + prob.q.size + prob.inflow.size +
                                                 prob.n_el * prob.n * 3 + 2 * prob.n_bnode)
    assert bench.option_flops_per_edg(2, 2, {"sigma"}) == 18 and bench.option_flops_per_edg(1, 2, {"fixup"}) == 0
    assert bench.shard_groups(64, 8, 7) == (56, 64) and bench.shard_groups(10, 3, 0) == (0, 4)
