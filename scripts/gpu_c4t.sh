for v in r4c4 r4c8 r8c8 r16c4 r8c2 r2c8; do for c in 4 3; do
SWEEP_LIB=build/$v.so timeout 120 python bench.py --config $c --no-e2e --no-cpu --steps 5 > gpurun_out/c4.json 2> gpurun_out/c4.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/c4.json').read().strip().splitlines()[-1]); print('$v C$c', round(d['roofline']['kernel_ms'],4))
except Exception as e: print('$v ERR', open('gpurun_out/c4.err').read()[-200:])
"
done; done
