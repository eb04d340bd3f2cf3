#!/bin/bash
# One GPU session: parity tests, benches, ncu launch list + full capture of the aggregation kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in teddy tsukuba; do timeout 600 python bench.py --config $c --steps 2000 --warmup 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config kitti --steps 300 --warmup 5 > gpurun_out/bench_kitti.json 2> gpurun_out/bench_kitti.err
timeout 600 python bench.py --config mb2014 --steps 10 --warmup 3 > gpurun_out/bench_mb2014.json 2> gpurun_out/bench_mb2014.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_teddy.csv python bench.py --steps 5 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_launch.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg -s 6 -c 2 -o gpurun_out/prof_teddy -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_full.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cost -s 6 -c 2 -o gpurun_out/prof_teddy_cost -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_cost.err
ls -la gpurun_out
