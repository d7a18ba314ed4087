timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "parity or regress or layout or debug or options" > gpurun_out/gputest11.txt 2>&1
B="--no-e2e --no-cpu --no-floors --steps 10"
for v in prod nosmemred; do
  L=""; [ "$v" != prod ] && L="--lib build/$v.so"
  for a in "--config 4" "--rank-of 8" "--rank-of 4" "--rank-of 2" "--config 5"; do
    t=$(echo $a | tr -d ' -')
    timeout 300 python bench.py $a $L $B > gpurun_out/sr_${v}_$t.json 2>/dev/null
  done
done
