OUT=gpurun_out; mkdir -p $OUT
timeout 300 ncu --section SourceCounters --section LaunchStats -k regex:"k_data|k_spec" -o $OUT/xcheck -f python tools/warp_sim_xcheck.py run > $OUT/xcheck_run.log 2>&1
tail -3 $OUT/xcheck_run.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_data -s 2 -c 1 -o $OUT/prof_C5d16_data -f python tools/prof_one.py C5d16 data 4 > $OUT/prof_C5d16_data.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_spec -s 2 -c 1 -o $OUT/prof_C5d16_spec -f python tools/prof_one.py C5d16 speculative 4 > $OUT/prof_C5d16_spec.log 2>&1
timeout 600 python bench.py > $OUT/bench_s5.json 2> $OUT/bench_s5.err; cat $OUT/bench_s5.json; tail -3 $OUT/bench_s5.err
