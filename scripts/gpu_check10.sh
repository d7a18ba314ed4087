set -x
timeout 900 python -m pytest tests/test_multirank_gloo.py tests/test_gpu_regress.py tests/test_gpu_debug.py -m gpu -x -q > gpurun_out/gputest_mr.txt 2>&1
for c in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
bash scripts/gpu_c5var.sh pa2 pa4
