mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "spec or appendix_a" > gpurun_out/t_triple.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_triple.log
for W in C5d14 C5d16 C5d18; do
  timeout 300 python tools/ab_geoms.py $W 'dict(variant=("spec_pred",))' --algo=speculative 2>&1 | tail -1
done
