# C5 kernel time of experiment builds (args: build names)
for v in "$@"; do
  timeout 300 python bench.py --lib build/$v.so --no-e2e --no-cpu --no-parity --steps 10 > gpurun_out/c5var_$v.json 2> gpurun_out/c5var_$v.err
done
timeout 300 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > gpurun_out/c5var_prod.json 2> gpurun_out/c5var_prod.err
