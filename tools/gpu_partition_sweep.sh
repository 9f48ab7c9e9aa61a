#!/bin/bash
# partition cost-model sweep on the p=512 C2-design fit (per-coordinate us)
mkdir -p gpurun_out
for cfg in "X=0" "GSS_PASS_W=0.05 GSS_ANY_W=0"; do
  echo "== $cfg" >> gpurun_out/psweep.txt
  env $cfg timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | tail -1 >> gpurun_out/psweep.txt
done
