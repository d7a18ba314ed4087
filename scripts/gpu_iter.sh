# quick iteration: new-kernel parity + C5 bench (both kernels) ; args: extra pytest -k filter
set -x
K=${1:-"many_group or dw_kernel or config5 or constant or beta or deterministic or recipe"}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_iter.log
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_dw.json 2> gpurun_out/bench_dw.err; echo bench=$?
SWEEP_KERNEL=classic timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_classic.json 2>&1; echo benchc=$?
python -c "
import json
for f in ['gpurun_out/bench_dw.json','gpurun_out/bench_classic.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'])
    except Exception as e: print(f, 'ERR', e)
"
