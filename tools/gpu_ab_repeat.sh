#!/bin/bash
# A/B with repeated processes (the run-to-run spread is per process): default vs each libfbs_exp*.so,
# interleaved, REPS times, Teddy.
mkdir -p gpurun_out; rm -f gpurun_out/rep_*
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/rep_tests.log 2>&1
for i in $(seq 1 ${REPS:-3}); do
  timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras > gpurun_out/rep_default_$i.json 2>/dev/null
  for v in paper_1807_02044_b200/libfbs_exp*.so; do
    n=$(basename $v .so); FBS_LIB=$PWD/$v timeout 300 python bench.py --steps 1000 --warmup 10 --no-extras > gpurun_out/rep_${n}_$i.json 2>/dev/null
  done
done
