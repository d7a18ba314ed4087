set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/c4full python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/c3full python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c3.log 2>&1
timeout 600 python scripts/shard_perf.py 8,16,32 "" 8 > gpurun_out/shard.txt 2>&1
