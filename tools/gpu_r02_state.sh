# round-2 re-entry: full GPU suite + bench (state check)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tail -1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -rf > gpurun_out/gputest.log 2>&1; echo tests=$?
tail -15 gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
