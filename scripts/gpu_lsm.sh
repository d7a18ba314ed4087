set -x
bash scripts/gpu_c5var.sh lsm
for k in 8 2; do timeout 300 python bench.py --lib build/lsm.so --rank-of $k --steps 10 --no-e2e --no-cpu > gpurun_out/lsm_rank$k.json 2> gpurun_out/lsm_rank$k.err; done
