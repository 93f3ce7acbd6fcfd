#!/usr/bin/env bash
# The paper's Table 1 structure on B200: the reference's
# bench flow (validation, warm-up, outer = alloc + H2D + kernel + D2H + free,
# inner = kernel, alloc) for the reference's CPU strategies and gpu-data /
# gpu-spec, on the paper's tree(11,16,19,7,1) over 65,536 and 16.8M records.
# Writes gpurun_out/table1_<M>.{json,txt}.  Run on a GPU box:
#     bash tools/table1.sh
set -euo pipefail
cd "$(dirname "$0")/.."
CLI=oracle/_ref/spectree_b200_cli
mkdir -p gpurun_out/t1
for M in 65536 16777216; do
  T=gpurun_out/t1/paper.json D=gpurun_out/t1/paper_$M.strec
  $CLI gen --depth 11 --leaves 16 --arity 19 --classes 7 --seed 1 --records $M --data-seed 2 \
      --out-tree $T --out-data $D
  S="--strategy serial --strategy data --strategy spec --strategy gpu-data --strategy gpu-spec"
  IT=$([ $M -gt 1000000 ] && echo 10 || echo 50)
  $CLI bench --tree $T --data $D $S --iterations $IT --warmup 3 --format json > gpurun_out/table1_$M.json
  $CLI bench --tree $T --data $D $S --iterations $IT --warmup 3 --format table > gpurun_out/table1_$M.txt
  rm -f $D
done
nproc > gpurun_out/table1_nproc.txt
