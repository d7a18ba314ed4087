# round-2 experiments: C5 layouts with two co-resident CTAs per SM, the 8-group rank's timeline and ncu capture
set -x
B="--no-e2e --no-cpu --no-floors --steps 10"
timeout 300 python bench.py $B > gpurun_out/v_prod.json 2> gpurun_out/v_prod.err
SWEEP_MAXWARPS=4 timeout 300 python bench.py --lib build/k4c4.so $B > gpurun_out/v_k4d8c4.json 2> gpurun_out/v_k4d8c4.err
SWEEP_CFG=4,8 SWEEP_MAXWARPS=4 timeout 300 python bench.py --lib build/k4c4.so $B > gpurun_out/v_k4g32c4.json 2> gpurun_out/v_k4g32c4.err
SWEEP_CFG=4,8 timeout 300 python bench.py --lib build/k4c4.so $B > gpurun_out/v_k4g32c4w8.json 2> gpurun_out/v_k4g32c4w8.err
SWEEP_CFG=2,16 timeout 300 python bench.py --lib build/k2c2m2.so $B > gpurun_out/v_k2c2m2.json 2> gpurun_out/v_k2c2m2.err
timeout 300 python bench.py --rank-of 8 $B > gpurun_out/v_r8.json 2> gpurun_out/v_r8.err
TRACE_SO=build/trace.so timeout 300 python profiles/trace_tasks.py 5 8 > gpurun_out/trace_r8.txt 2>&1
TRACE_SO=build/trace.so timeout 300 python profiles/trace_tasks.py 5 > gpurun_out/trace_c5.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/rank8 python bench.py --rank-of 8 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_rank8.log 2>&1
