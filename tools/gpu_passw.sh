for cfg in "GSS_BE_W=0" "GSS_BE_W=0.05 GSS_PASS_W=0" "GSS_BE_W=0.1 GSS_PASS_W=0" "GSS_BE_W=0.05" "GSS_BE_W=0.1"; do
  echo -n "$cfg: "; env $cfg timeout 600 python bench.py --c3-p 0 --no-c1 --c4 0 --c5 0 --no-cpu-baseline --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
