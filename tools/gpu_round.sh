# usage (on the GPU box): bash tools/gpu_round.sh [tests|trace|ncu|bench]...
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
for step in "$@"; do
case $step in
tests) timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 2>&1 | tail -8 ;;
trace) echo "trace: removed with the per-coordinate sweep";;
fit) timeout 300 python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 3 2>&1 | tail -3 ;;
api) timeout 300 python tools/prof_sweep.py --n 10000000 --p 64 --mode api --reps 50 2>&1 | tail -2 ;;
launches) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 70 -c 140 --csv \
    --log-file gpurun_out/launches.csv python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 3 \
    > gpurun_out/launches.log 2>&1; echo launches=$? ;;
ncu) timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 70 -c 1 \
    -o gpurun_out/prof_sweep python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 2 \
    > gpurun_out/ncu_full.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_full.log ;;
bench) timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?;
    tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json ;;
esac
done
