# time bench.py (C5, kernel only) for each build/<name>.so given as args
for v in "$@"; do
  timeout 300 python bench.py --lib build/$v.so --no-e2e --no-cpu --steps 5 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['roofline']['kernel_ms'],3), 'ms frac', round(d['roofline']['frac'],4))
except Exception as e: print('$v', 'ERR', open('gpurun_out/var_$v.err').read()[-300:])
"
done
