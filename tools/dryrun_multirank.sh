#!/bin/bash
# Dry run of bench.py's multi-rank logic with more ranks than GPUs (gloo; the JSON line
# carries "dry_run" and is not a measurement): frame sharding (teddy, kitti), row bands
# + gather (mb2014).  Usage (on a GPU box): bash tools/dryrun_multirank.sh [RANKS]
mkdir -p gpurun_out
n=${1:-2}
port=29611
for c in teddy kitti mb2014; do
  st=100; [ $c = mb2014 ] && st=5
  port=$((port + 1))
  FBS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus $n --config $c --steps $st --warmup 3 \
    > gpurun_out/dry_${c}_$n.json 2> gpurun_out/dry_${c}_$n.err
  echo "rc=$?" >> gpurun_out/dry_${c}_$n.err
done
