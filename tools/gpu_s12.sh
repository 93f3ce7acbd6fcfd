OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/clk_s12.txt
timeout 600 python tools/sweep.py --workload C2 --grid stages --iters 20 > $OUT/sweep_C2_stages.log 2>&1
grep BEST $OUT/sweep_C2_stages.log | cut -c1-600
