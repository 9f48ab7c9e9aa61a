# round-2 final evidence: ncu launch list of a bounded bench.py run, one full
# capture of the C2 cycle kernel (summarised into profiles/ncu_cycle_summary.json)
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02_bench_launches_final.csv python bench.py --steps 2 --warmup 3 --c4 0 --c5 0 \
  --no-c1 --no-cpu-baseline --no-parity --c3-cycles 1 > gpurun_out/r02_bench_under_ncu_final.log 2>&1; echo launches=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:cycle_kernel -s 2 -c 1 \
  -o gpurun_out/r02_prof_c2_final -f python tools/prof_sweep.py --n 10000000 --p 5000 --mode fit --cycles 2 \
  > gpurun_out/r02_ncu_c2_final.log 2>&1; echo ncu=$?; tail -2 gpurun_out/r02_ncu_c2_final.log
