set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "config1 or config2 or random or options or trt or debug or regress or 1d" > gpurun_out/gputest_1d.txt 2>&1
for c in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 600 python scripts/stress_parity.py 1500 43 > gpurun_out/stress.txt 2>&1
