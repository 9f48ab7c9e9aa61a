for d in 0 512; do GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 2 --model finegray 2>&1 | tail -1; done
timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -1
