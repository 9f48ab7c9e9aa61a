mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 1 -c 1 \
  -o gpurun_out/mask_new -f python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 2 > gpurun_out/mask_new.log 2>&1; echo new=$?
