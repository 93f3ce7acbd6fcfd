mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "appendix_a or slot_sizes or spec_window" > gpurun_out/t_g2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_g2.log
timeout 200 python tools/ab_geoms.py C1 'dict(group_lanes=2)' --algo=speculative --flush 2>&1 | tail -1
for W in C2 C5d16; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o gpurun_out/p_$W -f python tools/prof_one.py $W speculative 4 > /dev/null 2>&1; echo "ncu $W rc=$?"
  python tools/ncu_summary.py gpurun_out/p_$W.ncu-rep gpurun_out/ncu_${W}_speculative.json > /dev/null 2>&1
  python tools/ncu_sass_hot.py gpurun_out/p_$W.ncu-rep 30 > gpurun_out/ncu_${W}_speculative_hot.txt 2>&1; rm -f gpurun_out/p_$W.ncu-rep
done
