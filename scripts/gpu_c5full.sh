set -x
nproc > gpurun_out/c5full_test.txt
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config5_full_all_groups" --durations=3 >> gpurun_out/c5full_test.txt 2>&1
