set -x
timeout 300 python bench.py --config 3 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep1d_scan -s 3 -c 1 -o gpurun_out/c2scan python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_rows_kernel -s 3 -c 1 -o gpurun_out/c3rows python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c3rows.log 2>&1
timeout 300 python scripts/fault_repro.py build/hint.so > gpurun_out/fault_hint.txt 2>&1
