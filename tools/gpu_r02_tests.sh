# GPU tests + racecheck of the sanitizer cases (round 2)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gputest.log 2>&1; echo tests=$?
tail -8 gpurun_out/gputest.log
SAN_N=9000 SAN_GRID=2 timeout 900 compute-sanitizer --tool racecheck --print-limit 200 \
  python tools/sanitize_cases.py > gpurun_out/sanitize_racecheck.log 2>&1; echo racecheck=$?
grep -E "SUMMARY|Race reported" gpurun_out/sanitize_racecheck.log | sort | uniq -c | head -20
