for cfg in "" "4,8" "2,16" "4,4" "2,8" "1,16" "1,8"; do
  for mw in 8 4 2; do
  SWEEP_MAXWARPS=$mw SWEEP_CFG=$cfg timeout 120 python bench.py --config 4 --no-e2e --no-cpu --steps 5 > gpurun_out/c4.json 2> gpurun_out/c4.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/c4.json').read().strip().splitlines()[-1]); print('C4 cfg=$cfg maxwarps=$mw', round(d['roofline']['kernel_ms'],4))
except Exception as e: print('C4 $cfg ERR', open('gpurun_out/c4.err').read()[-200:])
"
  done
done
