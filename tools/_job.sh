GSS_DEBUG=256 timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 2 --model finegray 2>&1 | grep -v "^cycles" | tail -3 | cut -c1-400
echo "== free-running"; GSS_DEBUG=16 timeout 300 python tools/prof_sweep.py --n 10000000 --p 256 --mode fit --cycles 2 --model finegray 2>&1 | tail -1
echo "== tests"; timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
