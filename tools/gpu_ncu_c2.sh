# ncu evidence for the C2 cycle kernel (one CCD cycle = one launch)
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python tools/prof_sweep.py --n 10000000 --p 5000 \
  --mode fit --cycles 3 > gpurun_out/launches_c2.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 2 -c 1 \
  -o gpurun_out/prof_c2 python tools/prof_sweep.py --n 10000000 --p 5000 --mode fit --cycles 2 \
  > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_c2.log
