timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "many_group or dw_kernel or recipe or deterministic" > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_iter.log
bash scripts/gpu_variants.sh "$@"
