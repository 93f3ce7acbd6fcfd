mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "spec_window_formats or appendix_a or slot_sizes or fresh_tree" > gpurun_out/t_triple.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_triple.log
for W in C1 C3 C5d8 C5d12 C5d14 C5d16 C5d20; do
  F=""; [[ $W == C1 || $W == C3 ]] && F="--flush"
  timeout 300 python tools/ab_geoms.py $W 'dict(variant=("spec_quad",))' --algo=speculative $F 2>&1 | tail -1
done
