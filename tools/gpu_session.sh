#!/bin/bash
# One GPU session under gpurun: tests, bench, ncu launch list, ncu full captures.
#   gpurun --timeout 1800 -- 'bash tools/gpu_session.sh [tag] [parts]'
# parts: any of tests,bench,launches,ncu (default all)
TAG=${1:-r1}
PARTS=${2:-tests,bench,launches,ncu}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
if [[ $PARTS == *tests* ]]; then
  timeout 1200 python -m pytest tests -x -q -m gpu --durations=15 > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  tail -25 $OUT/pytest_gpu_$TAG.log
fi
if [[ $PARTS == *bench* ]]; then
  timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
  echo "bench rc=$?"; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
  timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref_$TAG.json 2>&1
  cat $OUT/bench_ref_$TAG.json | tail -1
fi
if [[ $PARTS == *launches* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --alt-steps 3 \
    --e2e-steps 1 --no-cpu-baseline > $OUT/launches_bench_$TAG.log 2>&1
  echo "launches rc=$?"
fi
if [[ $PARTS == *ncu* ]]; then
  for K in k_data k_spec; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o $OUT/prof_${K}_$TAG -f python bench.py --steps 3 --warmup 3 --alt-steps 3 --e2e-steps 1 \
      --no-cpu-baseline > $OUT/prof_${K}_$TAG.log 2>&1
    echo "ncu $K rc=$?"
  done
fi
ls -la $OUT
