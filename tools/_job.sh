for i in 1 2; do timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -1; done
