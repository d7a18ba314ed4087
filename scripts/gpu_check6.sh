set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config3 or random or layout" > gpurun_out/gputest_sub.txt 2>&1
for c in 3; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
export CUDA_ENABLE_COREDUMP_ON_EXCEPTION=1 CUDA_COREDUMP_FILE=gpurun_out/core_hint CUDA_COREDUMP_GENERATION_FLAGS='skip_nonrelocated_elf_images,skip_global_memory,skip_shared_memory,skip_local_memory,skip_constbank_memory'
timeout 300 python scripts/fault_repro.py build/hint.so > gpurun_out/fault_hint.txt 2>&1
unset CUDA_ENABLE_COREDUMP_ON_EXCEPTION
ls -la gpurun_out/core_hint* >> gpurun_out/fault_hint.txt 2>&1
if ls gpurun_out/core_hint* >/dev/null 2>&1; then
  timeout 300 cuda-gdb -batch -ex "target cudacore $(ls gpurun_out/core_hint* | head -1)" -ex "info cuda kernels" -ex "x/12i \$pc-96" -ex "info cuda lanes" > gpurun_out/fault_gdb.txt 2>&1
fi
