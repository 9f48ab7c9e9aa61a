for cfg in "GSS_PASS_W=0.05" "GSS_PASS_W=0.1" "GSS_PASS_W=0.15" "GSS_PASS_W=0.2" "GSS_PASS_W=0.1 GSS_BE_W=0.1" "GSS_PASS_W=0.15 GSS_BE_W=-0.1"; do
  echo -n "$cfg: "; env $cfg timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 2 2>&1 | tail -1
  env $cfg GSS_DEBUG=65536 timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 1 2>&1 | grep "gss cta" | awk '$NF>0{print $NF}' | sort -n | awk '{a[NR]=$1} END{print "   consume min",a[1],"median",a[int(NR/2)],"max",a[NR]}'
done
