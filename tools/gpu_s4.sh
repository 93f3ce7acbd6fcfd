OUT=gpurun_out; mkdir -p $OUT
for W in C5d12:1 C5d16:1 C3:32 C1:32; do
  N=${W%%:*}; T=${W##*:}
  timeout 400 python tools/sweep.py --workload $N --grid stages --tile $T --iters 10 > $OUT/sweep_${N}_s4.log 2>&1
done
timeout 300 ncu --section SourceCounters --section LaunchStats -k regex:"k_data|k_spec" -o $OUT/xcheck -f python tools/warp_sim_xcheck.py run > $OUT/xcheck_run.log 2>&1
tail -3 $OUT/xcheck_run.log
