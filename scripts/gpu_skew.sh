set -x
for k in 8 4; do
  timeout 300 python bench.py --lib build/skewlg.so --rank-of $k --steps 10 --no-e2e --no-cpu > gpurun_out/skew_rank$k.json 2> gpurun_out/skew_rank$k.err
done
timeout 300 python bench.py --lib build/skewlg.so --config 4 --steps 10 --no-e2e --no-cpu > gpurun_out/skew_c4.json 2> gpurun_out/skew_c4.err
