mkdir -p gpurun_out
timeout 300 python tools/trace_sweep.py --n 10000000 --p 16 2>&1 | head -6
timeout 120 python tools/prof_sweep.py --n 10000000 --p 64 --mode api --reps 50 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 5 -c 1 -o gpurun_out/prof_sweep2 python tools/prof_sweep.py --n 10000000 --p 64 --mode api --reps 3 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -2 gpurun_out/ncu_full.log
