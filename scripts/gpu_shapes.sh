# strip/chunk shape variants of the K <= 2 kernels (LL hand-off): 8-group rank, 16/32-group ranks, C4
B="--no-e2e --no-cpu --no-floors --no-parity --steps 10"
run() { timeout 300 python bench.py $2 $( [ "$1" != prod ] && echo --lib build/$1.so ) $B > gpurun_out/shp_$1_$(echo $2 | tr -d ' -').json 2>/dev/null; }
for v in prod r8t2 r8c8 r8t2c8; do run $v "--rank-of 8"; done
for v in prod k2t2 k2c8 k2t2c8; do run $v "--rank-of 4"; run $v "--rank-of 2"; done
for v in prod p1t2 p1c2 p1t8; do run $v "--config 4"; done
