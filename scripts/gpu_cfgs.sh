# classic kernel: lane-layout overrides (SWEEP_CFG=K,LG) and variant builds
export SWEEP_KERNEL=classic
for cfg in "4,16" "2,16" "2,32" "4,8" "1,32"; do
  SWEEP_CFG=$cfg timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/cfg.json 2> gpurun_out/cfg.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/cfg.json').read().strip().splitlines()[-1]); print('cfg $cfg', round(d['roofline']['kernel_ms'],3))
except Exception as e: print('cfg $cfg ERR', open('gpurun_out/cfg.err').read()[-300:])
"
done
bash scripts/gpu_variants.sh classic_c4
