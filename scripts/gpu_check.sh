# the -m gpu suite, smoke(), a bench line of every config, a random stress run
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in 5 4 3 2 1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
done
timeout 900 python scripts/stress_parity.py ${STRESS_N:-1500} 21 > gpurun_out/stress.txt 2>&1
