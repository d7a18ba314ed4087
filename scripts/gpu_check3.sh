set -x
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/gputest.txt 2>&1
for c in 1 2 3 4 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
timeout 900 python scripts/stress_parity.py 2000 23 > gpurun_out/stress.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/c5full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c5.log 2>&1
