# quick perf + correctness check of the cycle kernel (one GPU)
mkdir -p gpurun_out
timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -2
timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 3 --model finegray 2>&1 | tail -2
timeout 900 python -m pytest tests -x -q -m gpu --timeout 600 2>&1 | tail -4
