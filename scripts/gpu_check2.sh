set -x
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputest.txt 2>&1
for c in 1 2 3 4 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
for v in pc0; do timeout 300 python bench.py --lib build/$v.so --no-e2e --no-cpu --no-parity --steps 10 > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err; done
timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > gpurun_out/var_base.json 2> gpurun_out/var_base.err
timeout 900 python scripts/stress_parity.py 2000 22 > gpurun_out/stress.txt 2>&1
