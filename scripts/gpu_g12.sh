B="--no-e2e --no-cpu --no-floors --steps 10"
timeout 300 python bench.py --rank-of 4 $B > gpurun_out/lay_prod_r4.json 2>/dev/null
SWEEP_CFG=1,16 timeout 300 python bench.py --rank-of 4 --lib build/exp.so $B > gpurun_out/lay_116_r4.json 2>/dev/null
timeout 300 python bench.py --rank-of 2 $B > gpurun_out/lay_prod_r2.json 2>/dev/null
SWEEP_CFG=1,32 timeout 300 python bench.py --rank-of 2 --lib build/exp.so $B > gpurun_out/lay_132_r2.json 2>/dev/null
SWEEP_CFG=1,16 timeout 300 python bench.py --rank-of 2 --lib build/exp.so $B > gpurun_out/lay_116_r2.json 2>/dev/null
timeout 300 python bench.py --rank-of 8 $B > gpurun_out/lay_prod_r8.json 2>/dev/null
SWEEP_CFG=1,8 SWEEP_MAXWARPS=2 timeout 300 python bench.py --rank-of 8 --lib build/exp.so $B > gpurun_out/lay_18w2_r8.json 2>/dev/null
