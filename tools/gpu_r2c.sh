OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "appendix or spec or fresh" > $OUT/pytest_r2c.log 2>&1; tail -2 $OUT/pytest_r2c.log
timeout 600 python tools/read_floor.py > $OUT/read_floor_r2c.log 2>&1; cat $OUT/read_floor_r2c.log
for W in C1 C3; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_data -s 2 -c 1 -o $OUT/prof_${W}_data_r2c -f python tools/prof_one.py $W data 4 > /dev/null 2>&1; echo "ncu $W rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_forest -s 1 -c 1 -o $OUT/prof_C4_forest_r2c -f python tools/prof_forest.py > /dev/null 2>&1; echo "ncu C4 rc=$?"
