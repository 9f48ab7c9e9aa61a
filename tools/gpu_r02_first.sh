# round-2 first GPU pass: tests, bench, launch list, ncu full capture, sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 > gpurun_out/gputest.log 2>&1; echo tests=$?
tail -5 gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
for tool in memcheck racecheck synccheck; do
  SAN_N=9000 SAN_GRID=2 timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool=$?
  tail -4 gpurun_out/sanitize_$tool.log
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python tools/prof_sweep.py --n 10000000 --p 5000 --mode fit --cycles 2 \
  > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_c2.log
