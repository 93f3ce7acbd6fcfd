OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/clk_s13.txt
timeout 600 python -m pytest tests -x -q -m gpu -k "spec or ring or appendix" > $OUT/pytest_gpu_s13.log 2>&1; tail -1 $OUT/pytest_gpu_s13.log
for W in C2 C5d16; do timeout 400 python tools/sweep.py --workload $W --grid spec2 --iters 20 > $OUT/sweep_${W}_spec2c.log 2>&1; done
