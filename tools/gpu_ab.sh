# A/B: current libgss vs build/libgss_old.so (p=512 Cox, alternating)
for i in 1 2; do
  for d in 0 1; do
  echo -n "new dbg=$d: "; GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 $@ 2>&1 | tail -1
  echo -n "old dbg=$d: "; GSS_DEBUG=$d GSS_LIB=build/libgss_old.so timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 $@ 2>&1 | tail -1
  done
done
