# the many-group K = 4 layout (C5's) on the 32- and 16-group ranks, with 4- and 8-column chunks
B="--no-e2e --no-cpu --no-floors --steps 10"
timeout 300 python bench.py --rank-of 2 $B > gpurun_out/k4s_prod_r2.json 2>/dev/null
SWEEP_CFG=4,8 timeout 300 python bench.py --rank-of 2 --lib build/k4c4.so $B > gpurun_out/k4s_48c4_r2.json 2>/dev/null
SWEEP_CFG=4,8 timeout 300 python bench.py --rank-of 2 --lib build/k4c8x.so $B > gpurun_out/k4s_48c8_r2.json 2>/dev/null
timeout 300 python bench.py --rank-of 4 $B > gpurun_out/k4s_prod_r4.json 2>/dev/null
SWEEP_CFG=4,4 timeout 300 python bench.py --rank-of 4 --lib build/k4c4.so $B > gpurun_out/k4s_44c4_r4.json 2>/dev/null
SWEEP_CFG=4,4 timeout 300 python bench.py --rank-of 4 --lib build/k4c8x.so $B > gpurun_out/k4s_44c8_r4.json 2>/dev/null
