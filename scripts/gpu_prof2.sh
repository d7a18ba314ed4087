set -x
timeout 300 python bench.py --rank-of 8 --steps 10 --no-e2e --no-cpu > gpurun_out/bench_rank8.json 2> gpurun_out/bench_rank8.err
timeout 300 python bench.py --rank-of 4 --steps 10 --no-e2e --no-cpu > gpurun_out/bench_rank4.json 2> gpurun_out/bench_rank4.err
timeout 300 python bench.py --rank-of 2 --steps 10 --no-e2e --no-cpu > gpurun_out/bench_rank2.json 2> gpurun_out/bench_rank2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/rank8 python bench.py --rank-of 8 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_rank8.log 2>&1
