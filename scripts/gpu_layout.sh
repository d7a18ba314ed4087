# C4 / C3 / shard sweep times per lane layout (experiment build with SWEEP_CFG overrides)
set -x
for cfg in "" "4,8" "2,16" "4,4" "2,8"; do
  SWEEP_CFG=$cfg timeout 300 python bench.py --lib build/exp.so --config 4 --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/lay_c4_${cfg/,/x}.json 2> gpurun_out/lay_c4_${cfg/,/x}.err
done
timeout 300 python bench.py --config 4 --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/lay_c4_prod.json 2> gpurun_out/lay_c4_prod.err
SWEEP_SHARD_LIB=build/exp.so timeout 600 python scripts/shard_perf.py 8,16 ";4,2;2,4;4,4;2,8;1,8;1,16" 8 > gpurun_out/lay_shard.txt 2>&1
