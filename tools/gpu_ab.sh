#!/bin/bash
# A/B: default libfbs.so vs experimental variants (paper_1807_02044_b200/libfbs_exp*.so).
mkdir -p gpurun_out
for c in teddy kitti; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_default_$c.json 2>gpurun_out/ab_default_$c.err
  for v in paper_1807_02044_b200/libfbs_exp*.so; do
    n=$(basename $v .so); FBS_LIB=$PWD/$v timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_${n}_$c.json 2>gpurun_out/ab_${n}_$c.err
  done
done
