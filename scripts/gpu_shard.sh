# per-rank (group-sharded C5) sweep times for build/<lib>.so variants: args lib ...
for v in "$@"; do
  echo "== $v"
  SWEEP_SHARD_LIB=build/$v.so timeout 600 python scripts/shard_perf.py 8,16,32 ";1,8;1,16;2,8" 8,4,2 2>&1 | grep -v ERR
done
