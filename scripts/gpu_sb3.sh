for k in 8; do timeout 300 python bench.py --lib build/sb3.so --rank-of $k --steps 10 --no-e2e --no-cpu > gpurun_out/sb3_rank$k.json 2> gpurun_out/sb3_rank$k.err; done
