echo "== prof p=512"; GSS_DEBUG=256 timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 2>&1 | grep -v "^cycles" | tail -2 | cut -c1-400
echo "== no refresh"; timeout 300 python tools/prof_sweep.py --n 10000000 --p 512 --mode fit --cycles 3 --interval 1000000000 2>&1 | tail -1
echo "== tests"; timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
