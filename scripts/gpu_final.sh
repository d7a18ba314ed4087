# final round-1 evidence: smoke, bench lines (all configs + options + reference), ncu launch list and full capture
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
for c in 4 3 2 1; do python bench.py --config $c --no-cpu > gpurun_out/bench_c$c.json 2>> gpurun_out/bench_cfg.err; done
for o in sigma fixup halfrange trt; do python bench.py --no-cpu --no-e2e --opts $o > gpurun_out/bench_c5_$o.json 2>>gpurun_out/bench_opts.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/sweep2d_c5_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
