# Validate the N>1 bench path on a 1-GPU box: 2 ranks share cuda:0 over gloo
# (timing is meaningless -- both ranks contend for one GPU -- this checks the
# launch, barrier, max-over-ranks and single-JSON-line behaviour).
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 50 --warmup 3 --alt-steps 5 --e2e-steps 1 --backend gloo \
  > $OUT/bench_2rank.json 2> $OUT/bench_2rank.err; echo "rc=$?"; cat $OUT/bench_2rank.json | cut -c1-250; tail -3 $OUT/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29518 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > $OUT/bench_ref_2rank.json 2>&1; echo "rc=$?"; cat $OUT/bench_ref_2rank.json | grep impl | cut -c1-200
