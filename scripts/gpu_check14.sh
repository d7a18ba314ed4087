set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.txt 2>&1
for c in 2 4 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
