set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "config3 or config4 or config2 or config1 or layout or random or debug or regress" > gpurun_out/gputest_sub.txt 2>&1
for c in 2 3 4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
