for k in 8 4; do timeout 300 python bench.py --lib build/bps1.so --rank-of $k --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/bps1_rank$k.json 2> gpurun_out/bps1_rank$k.err; done
timeout 300 python bench.py --lib build/bps1.so --config 4 --steps 10 --no-e2e --no-cpu --no-parity > gpurun_out/bps1_c4.json 2> gpurun_out/bps1_c4.err
