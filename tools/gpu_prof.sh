#!/bin/bash
# ncu: full capture of the aggregation kernel (+ cost) at the Teddy config.
mkdir -p gpurun_out
tag=${1:-v}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg -s 2 -c 1 -o gpurun_out/prof_${tag}_agg -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_${tag}_agg.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cost -s 2 -c 1 -o gpurun_out/prof_${tag}_cost -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_${tag}_cost.err
