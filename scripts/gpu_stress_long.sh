# long random stress of the product against the oracle (several seeds)
for seed in 51 52 53 54 55; do timeout 1500 python scripts/stress_parity.py 20000 $seed > gpurun_out/stress_long_$seed.txt 2>&1; done
