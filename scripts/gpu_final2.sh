# round-2 closing evidence after the overlapped host copy: the -m gpu suite, smoke, bench lines
# (all configs + options + per-rank shards + reference arm), ncu launch list, a random stress run
timeout 2400 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/gputest_final2.txt 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/f2_bench_c5.json 2> gpurun_out/f2_bench_c5.err; echo bench5=$?
for c in 4 3 2 1; do python bench.py --config $c > gpurun_out/f2_bench_c$c.json 2>> gpurun_out/f2_bench_cfg.err; done
for o in sigma fixup halfrange trt; do python bench.py --no-cpu --no-parity --opts $o > gpurun_out/f2_bench_c5_$o.json 2>>gpurun_out/f2_bench_opts.err; done
for r in 2 4 8; do python bench.py --rank-of $r --no-cpu > gpurun_out/f2_bench_rank$r.json 2>>gpurun_out/f2_bench_rank.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/f2_bench_ref.json 2> gpurun_out/f2_bench_ref.err; echo ref=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/f2_ncu_l.log 2>&1; echo ncul=$?
timeout 900 python scripts/stress_parity.py ${STRESS_N:-4000} 43 > gpurun_out/f2_stress.txt 2>&1; echo stress=$?
