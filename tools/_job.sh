mkdir -p gpurun_out
echo "== tests"; timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_v9.json 2> gpurun_out/bench_v9.err; echo rc=$?
python -c "
import json
d=json.loads(open('gpurun_out/bench_v9.json').readline())
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['time_to_fit_s'], d['roofline']['frac'], d['secondary']['c3_finegray']['value'], d['secondary']['c3_finegray']['roofline']['frac'], d['clocks'])
"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; head -c 600 gpurun_out/bench_ref.json
