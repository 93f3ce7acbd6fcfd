mkdir -p gpurun_out
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize_run.py 8000 > gpurun_out/san_$T.log 2>&1; echo "$T rc=$?"; tail -3 gpurun_out/san_$T.log
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py --frames > gpurun_out/san_frames_memcheck.log 2>&1; echo "frames memcheck rc=$?"; tail -3 gpurun_out/san_frames_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py --frames > gpurun_out/san_frames_racecheck.log 2>&1; echo "frames racecheck rc=$?"; tail -3 gpurun_out/san_frames_racecheck.log
