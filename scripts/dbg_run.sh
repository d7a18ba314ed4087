for lib in build/nobck.so build/nopad.so build/both.so; do
 for shp in "9 6 2 10 32" "9 6 2 10 33"; do
  SWEEP_LIB=$lib timeout 60 python scripts/dbg_one.py $shp
 done
done
