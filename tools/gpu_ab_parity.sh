#!/bin/bash
# A/B: GPU parity + benches for the default libfbs.so and each libfbs_exp*.so.
mkdir -p gpurun_out; rm -f gpurun_out/ab_*
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab_default_tests.log 2>&1
for c in ${AB_CONFIGS:-teddy}; do
  timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_default_$c.json 2>gpurun_out/ab_default_$c.err
done
for v in paper_1807_02044_b200/libfbs_exp*.so; do
  [ -e "$v" ] || continue
  n=$(basename $v .so)
  [ -n "$AB_TESTS" ] && FBS_LIB=$PWD/$v timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/ab_${n}_tests.log 2>&1
  for c in ${AB_CONFIGS:-teddy}; do
    FBS_LIB=$PWD/$v timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras > gpurun_out/ab_${n}_$c.json 2>gpurun_out/ab_${n}_$c.err
  done
done
