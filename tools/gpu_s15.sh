OUT=gpurun_out; mkdir -p $OUT
timeout 600 python tools/sweep.py --workload C3 --grid regs1 --tile 32 --iters 10 > $OUT/sweep_C3_regs1.log 2>&1
timeout 600 python tools/sweep.py --workload C3 --grid regs1 --flush --iters 20 > $OUT/sweep_C3_regs1f.log 2>&1
