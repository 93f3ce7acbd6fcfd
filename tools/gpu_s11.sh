OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu -k "spec or ring or appendix or fuzz or exhaustive" > $OUT/pytest_gpu_s11.log 2>&1; tail -2 $OUT/pytest_gpu_s11.log
for W in C2 C5d8 C5d16; do
  timeout 400 python tools/sweep.py --workload $W --grid spec2 --iters 10 > $OUT/sweep_${W}_spec2b.log 2>&1
  grep '"samples_per_thread": 1' $OUT/sweep_${W}_spec2b.log | cut -c1-20 > /dev/null
done
