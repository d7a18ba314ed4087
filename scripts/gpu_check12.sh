set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "1-1 or 1-2 or dim1 or random or options or trt or debug or regress" > gpurun_out/gputest_1d.txt 2>&1
for c in 1 2; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
