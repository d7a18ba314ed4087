set -x
bash scripts/gpu_c5var.sh bp2
for k in 8 4 2; do timeout 300 python bench.py --lib build/bp2.so --rank-of $k --steps 10 --no-e2e --no-cpu > gpurun_out/bp2_rank$k.json 2> gpurun_out/bp2_rank$k.err; done
