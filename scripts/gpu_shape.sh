# per-rank (8-group shard) sweep time per strip/chunk shape of the K = 1 p = 2 kernel
for v in "$@"; do timeout 300 python bench.py --lib build/$v.so --rank-of 8 --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/shape_$v.json 2> gpurun_out/shape_$v.err; done
timeout 300 python bench.py --rank-of 8 --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/shape_prod.json 2> gpurun_out/shape_prod.err
