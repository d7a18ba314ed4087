set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.txt 2>&1
for c in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 python scripts/stress_parity.py 1500 25 > gpurun_out/stress.txt 2>&1
