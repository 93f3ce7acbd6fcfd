mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_flow.py -x -q -k "spec or appendix_a or pdl or order" > gpurun_out/t_pdl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_pdl.log
for W in C1 C3; do timeout 200 python tools/ab_geoms.py $W 'dict(pdl=3)' --algo=speculative --flush 2>&1 | tail -1; done
for W in C2 C5d12; do timeout 200 python tools/ab_geoms.py $W 'dict(pdl=3)' --algo=speculative 2>&1 | tail -1; done
