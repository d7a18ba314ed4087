for v in w4 w2; do timeout 300 python bench.py --lib build/$v.so --config 2 --steps 20 --no-e2e --no-cpu > gpurun_out/w_$v.json 2> gpurun_out/w_$v.err; done
timeout 300 python bench.py --config 2 --steps 20 --no-e2e --no-cpu > gpurun_out/w_prod.json 2> gpurun_out/w_prod.err
