set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python scripts/stress_parity.py 3000 41 > gpurun_out/stress.txt 2>&1
