set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench=$?
python bench.py --config 4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 2 -c 1 -o gpurun_out/sweep2d_c5 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
