SWEEP_LIB=build/pa2.so timeout 60 python scripts/dbg_one.py 13 7 2 8 64
bash scripts/gpu_full.sh
