GSS_DEBUG=256 timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | grep "prof cta" | tail -1 | cut -c150-420
