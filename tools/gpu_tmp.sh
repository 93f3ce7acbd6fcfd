mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "slot_sizes or appendix_a" > gpurun_out/t_half.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_half.log
for W in C1 C3; do timeout 200 python tools/ab_geoms.py $W 'dict(slot_records=1)' --algo=speculative --flush 2>&1 | tail -1; done
timeout 200 python tools/ab_geoms.py C3 'dict(slot_records=1)' --algo=speculative --tile=32 2>&1 | tail -1
for W in C5d8 C5d12 C5d20; do timeout 200 python tools/ab_geoms.py $W 'dict(slot_records=1)' --algo=speculative 2>&1 | tail -1; done
