# quick iteration: parity tests + A/B perf vs build/libgss_old.so (p=512 Cox)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --timeout 600 2>&1 | tail -4
for i in 1 2; do
  echo -n "new: "; timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -1
  echo -n "old: "; GSS_LIB=build/libgss_old.so timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -1
done
echo -n "new cprof: "; GSS_DEBUG=256 timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 2 2>&1 | grep -E "cprof" | tail -1
