# full GPU suite + C5/C4 kernel timings
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_full.log
for c in 5 4; do
timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 5 > gpurun_out/q$c.json 2> gpurun_out/q$c.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/q$c.json').read().strip().splitlines()[-1]); print('C$c', round(d['roofline']['kernel_ms'],3), 'ms', d['value'], 'frac', round(d['roofline']['frac'],4))
except Exception as e: print('C$c ERR', open('gpurun_out/q$c.err').read()[-500:])
"
done
