set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_r1c.log 2>&1; tail -3 $OUT/pytest_gpu_r1c.log
timeout 900 python tools/workloads.py --flush read > $OUT/workloads_read.log 2>&1; tail -3 $OUT/workloads_read.log
timeout 600 python tools/workloads.py --flush write --only C1,C3 > $OUT/workloads_write.log 2>&1
for W in C1 C3; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_data -s 2 -c 1 -o $OUT/prof_${W}_data -f python tools/prof_one.py $W data 4 > $OUT/prof_${W}_data.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o $OUT/prof_C2_spec -f python tools/prof_one.py C2 speculative 4 > $OUT/prof_C2_spec.log 2>&1
ls -la $OUT
