for lib in "" build/fixrolled.so; do
SWEEP_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --steps 3 --opts fixup > gpurun_out/fx.json 2> gpurun_out/fx.err
python -c "
import json
try:
    d=json.loads(open('gpurun_out/fx.json').read().strip().splitlines()[-1]); print('$lib fixup', round(d['roofline']['kernel_ms'],3))
except Exception as e: print('ERR', open('gpurun_out/fx.err').read()[-300:])
"
done
timeout 600 python -m pytest tests/test_gpu_options.py -q -x 2>&1 | tail -2
