GSS_DEBUG=65536 timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 1 2>&1 | grep "gss cta" | sort -t' ' -k3 -n > gpurun_out/spread.txt; wc -l gpurun_out/spread.txt
