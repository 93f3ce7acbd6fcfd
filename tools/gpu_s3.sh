OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_s3.log 2>&1; tail -2 $OUT/pytest_gpu_s3.log
for W in C2:1 C1:32 C3:32 C5d12:1 C5d16:1 C5d8:1; do
  N=${W%%:*}; T=${W##*:}
  timeout 300 python tools/sweep.py --workload $N --grid warps --tile $T --iters 10 > $OUT/sweep_${N}_s3.log 2>&1
  echo "== $N x$T"; grep BEST -A0 $OUT/sweep_${N}_s3.log | cut -c1-400
  grep '"samples_per_thread": 0, "blocks_per_sm": 0, "stages": 0, "warps_per_cta": 0' $OUT/sweep_${N}_s3.log | cut -c1-300
done
