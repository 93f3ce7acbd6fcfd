mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "appendix_a or exhaustive or fuzz" > gpurun_out/t_copies.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_copies.log
for W in C1 C3; do
  timeout 200 python tools/ab_geoms.py $W 'dict(tree_copies=2)' 'dict(tree_copies=4)' --flush 2>&1 | tail -1
done
timeout 200 python tools/ab_geoms.py C3 'dict(tree_copies=2)' 'dict(tree_copies=4)' --tile=32 2>&1 | tail -1
for W in C2 C5d8 C5d12 C5d16 C5d20; do
  timeout 200 python tools/ab_geoms.py $W 'dict(tree_copies=2)' 'dict(tree_copies=4)' 2>&1 | tail -1
done
