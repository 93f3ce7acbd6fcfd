OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -x -q -m gpu -k "stress or ring" > $OUT/pytest_gpu_s8.log 2>&1; tail -2 $OUT/pytest_gpu_s8.log
for W in C1 C3; do
  timeout 900 python tools/sweep.py --workload $W --grid small --flush --iters 20 > $OUT/sweep_${W}_small.log 2>&1; grep BEST -A8 $OUT/sweep_${W}_small.log | cut -c1-300
done
