mkdir -p gpurun_out
timeout 300 python tools/trace_cycle.py --n 10000000 --p 64 2>&1 | tail -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 2 -c 1 \
    -o gpurun_out/prof_cycle python tools/prof_sweep.py --n 10000000 --p 64 --mode fit --cycles 2 \
    > gpurun_out/ncu_cycle.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_cycle.log
