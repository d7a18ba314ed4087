for v in c4 c2; do for mw in 4 8; do
SWEEP_LIB=build/$v.so SWEEP_MAXWARPS=$mw timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/mw.json 2> gpurun_out/mw.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/mw.json').read().strip().splitlines()[-1]); print('$v maxwarps $mw', round(d['roofline']['kernel_ms'],3), 'ms total', round(d['ms_per_step'],3))
except Exception as e: print('$v $mw ERR', open('gpurun_out/mw.err').read()[-400:])
"
done; done
SWEEP_LIB=build/c4.so SWEEP_MAXWARPS=4 timeout 300 python scripts/dbg_one.py 33 5 2 8 130
SWEEP_LIB=build/c4.so SWEEP_MAXWARPS=4 timeout 300 python scripts/dbg_one.py 13 7 2 8 64
