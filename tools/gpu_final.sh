# Full evidence pass: GPU tests, bench + reference arm, launch list, ncu (C2 data/spec),
# workload table, C5 full sweep, CPU baselines.  Writes gpurun_out/*_fin.*
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu_$TAG.log 2>&1; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; cat $OUT/bench_$TAG.json | cut -c1-300
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref_$TAG.json 2>&1; tail -1 $OUT/bench_ref_$TAG.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 5 --warmup 3 --alt-steps 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_data -s 2 -c 1 -o $OUT/prof_C2_data_$TAG -f python tools/prof_one.py C2 data 4 > $OUT/prof_C2_data_$TAG.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o $OUT/prof_C2_spec_$TAG -f python tools/prof_one.py C2 speculative 4 > $OUT/prof_C2_spec_$TAG.log 2>&1
timeout 1200 python tools/workloads.py --flush read > $OUT/workloads_$TAG.log 2>&1; tail -1 $OUT/workloads_$TAG.log | cut -c1-200
timeout 1200 python tools/c5_sweep.py --gpus 1 > $OUT/c5_sweep_$TAG.log 2>&1; tail -1 $OUT/c5_sweep_$TAG.log | cut -c1-200
ls $OUT | wc -l
# per-config captures of the data kernel (C1 / C3 small-input paths, C5 d16 deep tree)
for W in C1 C3 C5d16; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_data -s 2 -c 1 -o $OUT/prof_${W}_data_$TAG -f python tools/prof_one.py $W data 4 > $OUT/prof_${W}_data_$TAG.log 2>&1
done
ls $OUT | wc -l
# compute-sanitizer over every kernel family (small launches)
mkdir -p $OUT/san
for T in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $T python tools/sanitize_run.py 3000 > $OUT/san/r1_$T.log 2>&1; echo "$T rc=$?"
done
