# final round evidence: the -m gpu suite, smoke, bench lines (all configs + options + reference + per-rank
# shards), 20k-case stress, ncu launch list and full captures (C5, C4, the 8-group rank), shard times
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gputest_final.txt 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
for c in 4 3 2 1; do python bench.py --config $c > gpurun_out/bench_c$c.json 2>> gpurun_out/bench_cfg.err; done
for o in sigma fixup halfrange trt; do python bench.py --no-cpu --no-e2e --no-parity --opts $o > gpurun_out/bench_c5_$o.json 2>>gpurun_out/bench_opts.err; done
for r in 2 4 8; do python bench.py --rank-of $r --no-cpu --no-e2e > gpurun_out/bench_rank$r.json 2>>gpurun_out/bench_rank.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 1500 python scripts/stress_parity.py 20000 41 > gpurun_out/stress20k.txt 2>&1; echo stress=$?
timeout 600 python scripts/shard_perf.py 8,16,32 "" 8 > gpurun_out/shard.txt 2>&1
timeout 300 python scripts/ll_check.py 4 > gpurun_out/llcheck_c4.txt 2>&1
timeout 300 python scripts/ll_check.py 5 8 > gpurun_out/llcheck_r8.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_l.log 2>&1; echo ncul=$?
ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/sweep2d_c5_final python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/sweep2d_c4_final python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_c4.log 2>&1; echo ncuc4=$?
ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/sweep2d_r8_final python bench.py --rank-of 8 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_r8.log 2>&1; echo ncur8=$?
