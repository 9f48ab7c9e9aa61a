for d in 0 16 1; do
  echo -n "FG dbg=$d: "; GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 2 --model finegray 2>&1 | tail -1
done
GSS_DEBUG=256 timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 2 --model finegray 2>&1 | grep "gss prof" | tail -1
