timeout 300 python scripts/dbg_one.py 13 7 2 8 64; timeout 300 python scripts/dbg_one.py 33 5 2 8 130
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
for v in "" classic; do
SWEEP_KERNEL=$v timeout 300 python bench.py --no-e2e --no-cpu --steps 5 > gpurun_out/q5.json 2> gpurun_out/q5.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/q5.json').read().strip().splitlines()[-1]); print('C5 $v', round(d['roofline']['kernel_ms'],3), 'ms', d['value'], 'frac', round(d['roofline']['frac'],4))
except Exception as e: print('C5 ERR', open('gpurun_out/q5.err').read()[-500:])
"
done
