#!/bin/bash
# per-tile features + per-CTA consume times for fitting the partition cost model
mkdir -p gpurun_out/tilecost
for P in 512 5000; do
for cfg in "GSS_PASS_W=0.04" "GSS_PASS_W=0 GSS_ANY_W=0"; do
  tag=$(echo "p${P}_$cfg" | tr ' =' '__')
  env $cfg GSS_DEBUG=65536 GSS_TILE_DUMP=1 GSS_VERBOSE=1 timeout 400 python tools/prof_sweep.py --n 10000000 --p $P --mode fit --cycles 2 \
     > gpurun_out/tilecost/$tag.out 2> gpurun_out/tilecost/$tag.err
  tail -1 gpurun_out/tilecost/$tag.out
done
done
