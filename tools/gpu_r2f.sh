# Round-2 evidence refresh: workloads table, C5 and C4 bench lines, C2 bench + reference arm, launch list, ncu C2 data/spec
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 1200 python bench.py --workload C5 --steps 20 --warmup 3 > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err; echo "c5 rc=$?"
timeout 900 python bench.py --workload C4 --steps 20 --warmup 3 > $OUT/bench_c4_$TAG.json 2> $OUT/bench_c4_$TAG.err; echo "c4 rc=$?"
timeout 600 python bench.py --workload PAPER --steps 200 --warmup 5 > $OUT/bench_paper_$TAG.json 2> $OUT/bench_paper_$TAG.err; echo "paper rc=$?"
timeout 1200 python tools/workloads.py --flush read > $OUT/workloads_$TAG.log 2>&1; echo "work rc=$?"
cp $OUT/workloads_read.json $OUT/workloads_$TAG.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --alt-steps 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1; echo "launch rc=$?"
for A in data speculative; do K=k_data; [[ $A == speculative ]] && K=k_spec
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/prof_C2_${A}_$TAG -f \
    python tools/prof_one.py C2 $A 4 > /dev/null 2>&1; echo "ncu C2 $A rc=$?"; done
