mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_frames.py -x -q > gpurun_out/t_frames.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_frames.log
for RB in "8 4" "8 1" "4 1" "16 8"; do set -- $RB
timeout 100 python tools/frames_bench.py --ring $1 --pub-batch $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ring',$1,'batch',$2, {k: round(d[k]['us_per_frame'],2) for k in ('single','batched','stream')})"
done
