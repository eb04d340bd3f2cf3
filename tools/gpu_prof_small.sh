#!/bin/bash
mkdir -p gpurun_out
tag=${1:-v}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cost -s 2 -c 1 -o gpurun_out/prof_${tag}_cost -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_${tag}_cost.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 2 -c 1 -o gpurun_out/prof_${tag}_fin -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_${tag}_fin.err
