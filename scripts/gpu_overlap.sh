# sweep_run_host's overlapped copy: its tests, then bench lines (e2e) of C5 / C4 / the 8-group rank
set -x
timeout 900 python -m pytest tests/test_gpu_regress.py tests/test_gpu_parity.py -x -q -k "overlapped or host or ll_ring" > gpurun_out/ov_tests.txt 2>&1; echo tests=$?
timeout 600 python bench.py --no-cpu > gpurun_out/ov_bench_c5.json 2> gpurun_out/ov_bench_c5.err; echo b5=$?
timeout 600 python bench.py --config 4 --no-cpu > gpurun_out/ov_bench_c4.json 2> gpurun_out/ov_bench_c4.err; echo b4=$?
timeout 600 python bench.py --config 3 --no-cpu > gpurun_out/ov_bench_c3.json 2> gpurun_out/ov_bench_c3.err; echo b3=$?
