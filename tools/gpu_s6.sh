OUT=gpurun_out; mkdir -p $OUT
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py 3000 > $OUT/sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -4 $OUT/sanitize_$T.log
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o $OUT/prof_C2_spec_r1e -f python tools/prof_one.py C2 speculative 4 > $OUT/prof_C2_spec_r1e.log 2>&1; tail -2 $OUT/prof_C2_spec_r1e.log
timeout 900 python tools/cpu_baselines.py > $OUT/cpu_baselines.log 2>&1; tail -2 $OUT/cpu_baselines.log
timeout 1200 python tools/c5_sweep.py --gpus 1 > $OUT/c5_sweep.log 2>&1; tail -9 $OUT/c5_sweep.log
