#!/bin/bash
# Round-2 (session 3) evidence: GPU tests, smoke, bench lines (C2 + reference
# arm, C5, C4, PAPER), workload table, frame stream, launch list, ncu of the
# speculative lane-triple kernels.
#   gpurun --timeout 3000 -- 'bash tools/gpu_r2s3.sh TAG [parts]'
TAG=${1:-r2s3}
PARTS=${2:-tests,bench,c5,c4,paper,work,frames,launch,ncu}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu_$TAG.txt 2>&1
if [[ $PARTS == *tests* ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
fi
if [[ $PARTS == *bench* ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
  timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
fi
[[ $PARTS == *c5* ]] && { timeout 1200 python bench.py --workload C5 --steps 20 --warmup 3 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err; echo "c5 rc=$?"; }
[[ $PARTS == *c4* ]] && { timeout 900 python bench.py --workload C4 --steps 20 --warmup 3 > $OUT/bench_c4_$TAG.json 2> $OUT/bench_c4_$TAG.err; echo "c4 rc=$?"; }
[[ $PARTS == *paper* ]] && { timeout 600 python bench.py --workload PAPER --steps 200 --warmup 5 > $OUT/bench_paper_$TAG.json 2> $OUT/bench_paper_$TAG.err; echo "paper rc=$?"; }
if [[ $PARTS == *work* ]]; then
  timeout 1200 python tools/workloads.py --flush read > $OUT/workloads_$TAG.log 2>&1; echo "work rc=$?"
  cp $OUT/workloads_read.json $OUT/workloads_$TAG.json 2>/dev/null
fi
[[ $PARTS == *frames* ]] && { timeout 120 python tools/frames_bench.py > $OUT/frames_$TAG.log 2>&1; echo "frames rc=$?"; cp $OUT/frames_C3.json $OUT/frames_C3_$TAG.json; }
if [[ $PARTS == *launch* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --alt-steps 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launch rc=$?"
fi
if [[ $PARTS == *ncu* ]]; then
  # reports are summarised on the box (gpurun_out must stay < 64 MiB)
  for WA in ${NCU_LIST:-C5d12:speculative C5d20:speculative C1:speculative C3:speculative C3:data C5d12:data}; do
    W=${WA%%:*}; A=${WA##*:}; K=k_data; [[ $A == speculative ]] && K=k_spec
    R=$OUT/prof_${W}_${A}_$TAG
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $R -f \
      python tools/prof_one.py $W $A 4 > $R.log 2>&1; echo "ncu $W $A rc=$?"
    python tools/ncu_summary.py $R.ncu-rep $OUT/ncu_${W}_${A}_$TAG.json > /dev/null 2>&1
    python tools/ncu_sass_hot.py $R.ncu-rep 30 > $OUT/ncu_${W}_${A}_${TAG}_hot.txt 2>&1
    rm -f $R.ncu-rep
  done
fi
if [[ $PARTS == *forest* ]]; then
  R=$OUT/prof_C4_forest_$TAG
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forest -s 1 -c 1 -o $R -f \
    python tools/prof_forest.py > $R.log 2>&1; echo "ncu C4 rc=$?"
  python tools/ncu_summary.py $R.ncu-rep $OUT/ncu_C4_forest_$TAG.json > /dev/null 2>&1
  python tools/ncu_sass_hot.py $R.ncu-rep 30 > $OUT/ncu_C4_forest_${TAG}_hot.txt 2>&1
  rm -f $R.ncu-rep
fi
ls $OUT | wc -l
