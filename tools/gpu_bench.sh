# usage: bash tools/gpu_bench.sh [full]
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 240 2>&1 | tail -5
timeout 120 python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 3 2>&1 | tail -3
timeout 120 python tools/prof_sweep.py --n 10000000 --p 64 --mode api --reps 50 2>&1 | tail -2
if [ "$1" = full ]; then
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo rc=$?
tail -5 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
fi
