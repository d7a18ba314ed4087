# A/B of the product against HEAD and experiment builds: bench lines of C5, C4 and the 8-group rank
# (usage: bash scripts/gpu_ab.sh build1 build2 ...; names of build/<name>.so)
B="--no-e2e --no-cpu --no-floors --steps 10"
for v in prod "$@"; do
  L=""; [ "$v" != prod ] && L="--lib build/$v.so"
  for a in "--config 5" "--config 4" "--rank-of 8"; do
    t=$(echo $a | tr -d ' -')
    timeout 300 python bench.py $a $L $B > gpurun_out/ab_${v}_$t.json 2> gpurun_out/ab_${v}_$t.err
  done
done
