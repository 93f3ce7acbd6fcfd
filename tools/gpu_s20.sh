OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_s20.log 2>&1; tail -2 $OUT/pytest_gpu_s20.log
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 10 python tools/sanitize_run.py 3000 > $OUT/sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -2 $OUT/sanitize_$T.log
done
