#!/bin/bash
# C4 time-to-result vs fits per batched launch (GSS_BATCH_MAX)
mkdir -p gpurun_out
for b in "$@"; do
  echo "== GSS_BATCH_MAX=$b" >> gpurun_out/c4b.txt
  GSS_BATCH_MAX=$b GSS_CV_VERBOSE=1 timeout 600 python tools/c4_cv.py 2>> gpurun_out/c4b.txt | grep -o '"time_to_result_s": [0-9.]*' >> gpurun_out/c4b.txt
done
