for d in 65537; do
GSS_DEBUG=$d timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 1 2>&1 | grep "gss cta" | awk '$NF>0' | sort -t' ' -k3 -n > gpurun_out/spread_$d.txt
done
