B="--no-e2e --no-cpu --no-floors --no-parity --steps 10"
for rep in 1 2; do
for v in prod nobal nobalng; do
  L=""; [ "$v" != prod ] && L="--lib build/$v.so"
  for a in "--config 5" "--config 4" "--rank-of 8" "--rank-of 4"; do
    t=$(echo $a | tr -d ' -')
    timeout 300 python bench.py $a $L $B > gpurun_out/bal_${v}_${t}_$rep.json 2>/dev/null
  done
done
done
