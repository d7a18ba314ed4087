set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep2d_rows_kernel -s 3 -c 1 -o gpurun_out/c3rows python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_c3rows.log 2>&1
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
export CUDA_ENABLE_COREDUMP_ON_EXCEPTION=1 CUDA_COREDUMP_FILE=gpurun_out/core_hint CUDA_COREDUMP_GENERATION_FLAGS='skip_nonrelocated_elf_images,skip_global_memory,skip_shared_memory,skip_local_memory'
timeout 300 python scripts/fault_repro.py build/hint.so > gpurun_out/fault_hint.txt 2>&1
unset CUDA_ENABLE_COREDUMP_ON_EXCEPTION CUDA_COREDUMP_GENERATION_FLAGS
ls -la gpurun_out/ >> gpurun_out/fault_hint.txt 2>&1
c=$(ls gpurun_out/core_hint* 2>/dev/null | head -1)
if [ -n "$c" ]; then timeout 300 cuda-gdb -batch -ex "target cudacore $c" -ex "info cuda kernels" -ex "x/16i \$pc-128" -ex "info cuda lanes" > gpurun_out/fault_gdb.txt 2>&1; fi
