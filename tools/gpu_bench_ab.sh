#!/bin/bash
# C2/C3 bench lines under two partition cost models (new default vs round-2 default)
mkdir -p gpurun_out
python bench.py --no-cpu-baseline --no-c1 --c4 0 --c5 0 --no-parity > gpurun_out/bab_new.json 2> gpurun_out/bab_new.err
GSS_PASS_W=0.05 GSS_ANY_W=0 python bench.py --no-cpu-baseline --no-c1 --c4 0 --c5 0 --no-parity > gpurun_out/bab_old.json 2> gpurun_out/bab_old.err
python bench.py --no-cpu-baseline --no-c1 --c4 0 --c5 0 --no-parity > gpurun_out/bab_new2.json 2> gpurun_out/bab_new2.err
