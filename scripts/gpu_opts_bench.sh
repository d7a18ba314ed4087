for o in sigma halfrange trt fixup; do python bench.py --no-cpu --no-e2e --opts $o --steps 5 > gpurun_out/bench_c5_$o.json 2>>gpurun_out/bench_opts.err; tail -1 gpurun_out/bench_c5_$o.json | cut -c1-400; done
tail -5 gpurun_out/bench_opts.err
