#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/ab_*
timeout 300 python bench.py --config teddy --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_default_teddy.json 2>gpurun_out/ab_default_teddy.err
for v in paper_1807_02044_b200/libfbs_exp*.so; do
  n=$(basename $v .so); FBS_LIB=$PWD/$v timeout 300 python bench.py --config teddy --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_${n}_teddy.json 2>gpurun_out/ab_${n}_teddy.err
done
