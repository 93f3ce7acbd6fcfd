OUT=gpurun_out; mkdir -p $OUT
for W in C5d12 C5d16; do for A in speculative data; do
  K=k_data; [[ $A == speculative ]] && K=k_spec
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o $OUT/prof_${W}_${A}_r2b -f \
      python tools/prof_one.py $W $A 4 > $OUT/prof_${W}_${A}_r2b.log 2>&1; echo "ncu $W $A rc=$?"
done; done
