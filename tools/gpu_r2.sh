#!/bin/bash
# Round-2 evidence session on one B200:
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2.sh TAG [parts]'
# parts: tests,smoke,bench,multi,c5,work,launch,ncu (default: all but ncu)
TAG=${1:-r2}
PARTS=${2:-tests,smoke,bench,multi,c5,work,launch}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > $OUT/gpu_$TAG.txt 2>&1
nproc >> $OUT/gpu_$TAG.txt
if [[ $PARTS == *tests* ]]; then
  timeout 1500 python -m pytest tests -x -q -m gpu --durations=20 > $OUT/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
fi
if [[ $PARTS == *smoke* ]]; then
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
fi
if [[ $PARTS == *bench* ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
  echo "bench rc=$?"; cut -c1-600 $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
  timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
  echo "ref rc=$?"; tail -1 $OUT/bench_ref_$TAG.json | cut -c1-300
fi
if [[ $PARTS == *multi* ]]; then
  timeout 900 python bench.py --gpus 2 --steps 50 --warmup 3 > $OUT/bench_g2_$TAG.json 2> $OUT/bench_g2_$TAG.err
  echo "g2 rc=$?"; cut -c1-400 $OUT/bench_g2_$TAG.json; tail -3 $OUT/bench_g2_$TAG.err
fi
if [[ $PARTS == *c5* ]]; then
  timeout 1500 python bench.py --workload C5 --steps 20 --warmup 3 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err
  echo "c5 rc=$?"; cut -c1-600 $OUT/bench_c5_$TAG.json; tail -3 $OUT/bench_c5_$TAG.err
fi
if [[ $PARTS == *work* ]]; then
  timeout 1200 python tools/workloads.py --flush read > $OUT/workloads_$TAG.log 2>&1; echo "work rc=$?"; tail -1 $OUT/workloads_$TAG.log | cut -c1-300
fi
if [[ $PARTS == *launch* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --alt-steps 3 --e2e-steps 1 --no-cpu-baseline > $OUT/launches_bench_$TAG.log 2>&1
  echo "launch rc=$?"
fi
if [[ $PARTS == *ncu* ]]; then
  for W in C1 C3 C5d16 C2; do for A in data speculative; do
    K=k_data; [[ $A == speculative ]] && K=k_spec
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/prof_${W}_${A}_$TAG -f \
      python tools/prof_one.py $W $A 4 > $OUT/prof_${W}_${A}_$TAG.log 2>&1; echo "ncu $W $A rc=$?"
  done; done
fi
ls $OUT | wc -l
