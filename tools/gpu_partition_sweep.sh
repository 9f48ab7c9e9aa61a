#!/bin/bash
# partition cost-model sweep on a CCD fit (per-coordinate us); P = columns
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "== $cfg p=${P:-512}" >> gpurun_out/psweep.txt
  env $cfg timeout 300 python tools/prof_sweep.py --n 10000000 --p ${P:-512} --mode fit --cycles ${CYC:-3} --model ${MODEL:-cox} 2>&1 | tail -1 >> gpurun_out/psweep.txt
done
