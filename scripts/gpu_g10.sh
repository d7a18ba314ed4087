B="--no-e2e --no-cpu --no-floors --no-parity --steps 10"
for v in prod ablrelax ablnowait; do
  L=""; [ "$v" != prod ] && L="--lib build/$v.so"
  for a in "--config 5" "--rank-of 2"; do
    t=$(echo $a | tr -d ' -')
    timeout 300 python bench.py $a $L $B > gpurun_out/abl_${v}_${t}.json 2>/dev/null
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/c4_ll python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_kernel -s 3 -c 1 -o gpurun_out/r8_ll python bench.py --rank-of 8 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity --no-floors > gpurun_out/ncu_r8.log 2>&1
