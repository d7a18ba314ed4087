# kernel time of configs C3, C4 and the C5 per-rank shards (G_loc = 8, 16) for build/<lib>.so variants
for v in "$@"; do
  for c in 3 4; do
    timeout 300 python bench.py --lib build/$v.so --config $c --no-e2e --no-cpu --steps 20 > gpurun_out/cf_${v}_$c.json 2> gpurun_out/cf_${v}_$c.err
    python -c "
import json
try:
    d=json.loads(open('gpurun_out/cf_${v}_$c.json').read().strip().splitlines()[-1]); print('$v C$c', round(d['roofline']['kernel_ms'],4), 'ms step', round(d['ms_per_step'],4))
except Exception as e: print('$v C$c ERR', open('gpurun_out/cf_${v}_$c.err').read()[-300:])
"
  done
  SWEEP_SHARD_LIB=build/$v.so timeout 300 python scripts/shard_perf.py 8,16 "" 8 2>&1 | sed "s/^/$v /"
done
