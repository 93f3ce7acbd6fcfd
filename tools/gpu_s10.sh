OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_s10.log 2>&1; tail -2 $OUT/pytest_gpu_s10.log
for W in C2 C5d8 C5d12 C5d16 C5d20; do
  timeout 400 python tools/sweep.py --workload $W --grid spec2 --iters 10 > $OUT/sweep_${W}_spec2.log 2>&1
done
timeout 300 python tools/sweep.py --workload C3 --grid spec2 --tile 32 --iters 5 > $OUT/sweep_C3_spec2.log 2>&1
