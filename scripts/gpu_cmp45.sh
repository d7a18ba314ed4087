for v in "$@"; do for c in 5 4 3; do
timeout 120 python bench.py --lib build/$v.so --config $c --no-e2e --no-cpu --steps 5 > gpurun_out/cx.json 2> gpurun_out/cx.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/cx.json').read().strip().splitlines()[-1]); print('$v C$c', round(d['roofline']['kernel_ms'],4))
except Exception as e: print('$v ERR', open('gpurun_out/cx.err').read()[-200:])
"
done; done
