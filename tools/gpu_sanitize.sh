# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  SAN_N=9000 SAN_GRID=2 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_${tool}_r02_final.log 2>&1; echo $tool=$?
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|cases done|Error|error" gpurun_out/sanitize_${tool}_r02_final.log | tail -4
done
