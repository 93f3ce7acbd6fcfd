OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_s9.log 2>&1; tail -2 $OUT/pytest_gpu_s9.log
timeout 600 python tools/sweep.py --workload C3 --grid regs --tile 32 --iters 10 > $OUT/sweep_C3_regs.log 2>&1
timeout 600 python tools/sweep.py --workload C3 --grid regs --flush --iters 20 > $OUT/sweep_C3_regs_flush.log 2>&1
timeout 600 python tools/sweep.py --workload C1 --grid small --flush --iters 20 > $OUT/sweep_C1_small2.log 2>&1
grep -h BEST -A3 $OUT/sweep_C3_regs.log $OUT/sweep_C3_regs_flush.log | cut -c1-200
