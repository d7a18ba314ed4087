# time the C5 fixup option (kernel only) for build/<lib>.so under SWEEP_CFG layouts: args lib:cfg ...
for spec in "$@"; do
  lib=${spec%%:*}; cfg=${spec#*:}; tag=${lib}_${cfg/,/x}
  SWEEP_CFG=$cfg timeout 300 python bench.py --lib build/$lib.so --no-e2e --no-cpu --steps 5 --opts fixup > gpurun_out/fx_$tag.json 2> gpurun_out/fx_$tag.err
  python -c "
import json
try:
    d=json.loads(open('gpurun_out/fx_$tag.json').read().strip().splitlines()[-1]); print('$tag', round(d['roofline']['kernel_ms'],3), 'ms', d['ms_per_step'])
except Exception as e: print('$tag', 'ERR', open('gpurun_out/fx_$tag.err').read()[-300:])
"
done
