# per-rank sweep time of the 8- and 16-group shards of C5 for build/<lib>.so variants
for v in "$@"; do
  SWEEP_SHARD_LIB=build/$v.so timeout 300 python scripts/shard_perf.py 8,16 "" 8 2>&1 | grep -v Traceback | sed "s/^/$v /" | cut -c1-110
done
