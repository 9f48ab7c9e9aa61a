for d in 1 16 0; do
  for v in "GSS_X=1" "GSS_NO_COMPACT=1"; do
  echo -n "dbg=$d $v: "; env $v GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 2 2>&1 | tail -1
  done
  echo -n "dbg=$d old: "; GSS_LIB=build/libgss_old.so GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 2 2>&1 | tail -1
done
