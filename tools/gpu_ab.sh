#!/bin/bash
# A/B of library variants / GSS_DEBUG bits on a CCD fit (per-coordinate us):
#   P=5000 bash tools/gpu_ab.sh default:0 build/exp/libgss.so:0 default:2097152 ...
set -u
mkdir -p gpurun_out
for vd in "$@"; do
  v=${vd%%:*}; d=${vd##*:}
  echo "== $v dbg=$d p=${P:-512} ${MODEL:-cox}" >> gpurun_out/ab.txt
  if [ "$v" = default ]; then unset GSS_LIB; else export GSS_LIB=$PWD/$v; fi
  GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p ${P:-512} --mode fit --cycles ${CYC:-3} --model ${MODEL:-cox} 2>&1 | tail -2 >> gpurun_out/ab.txt
done
