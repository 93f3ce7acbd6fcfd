OUT=gpurun_out; mkdir -p $OUT
for W in C5d12 C5d16 C5d20 C5d8; do
  timeout 600 python tools/sweep.py --workload $W --grid regs1+regs0 --iters 10 > $OUT/sweep_${W}_regs1.log 2>&1
done
timeout 600 python tools/sweep.py --workload C1 --grid regs1+regs0 --flush --iters 20 > $OUT/sweep_C1_regs1f.log 2>&1
timeout 600 python tools/sweep.py --workload C2 --grid regs0 --iters 10 > $OUT/sweep_C2_regs0.log 2>&1
