OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_s7.log 2>&1; tail -2 $OUT/pytest_gpu_s7.log
for i in 1 2 3; do
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o $OUT/prof_C2_spec_s7_$i -f python tools/prof_one.py C2 speculative 4 > $OUT/prof_C2_spec_s7_$i.log 2>&1; tail -2 $OUT/prof_C2_spec_s7_$i.log
done
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py 3000 > $OUT/sanitize_racecheck_s7.log 2>&1; tail -3 $OUT/sanitize_racecheck_s7.log
timeout 1200 python tools/c5_sweep.py --gpus 1 > $OUT/c5_sweep.log 2>&1; tail -9 $OUT/c5_sweep.log | cut -c1-400
