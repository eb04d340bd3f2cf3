#!/bin/bash
# One GPU session for the record: parity, smoke, benches (all configs), reference arm,
# ncu launch list + full captures of the two main kernels at the headline config.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_teddy.json 2> gpurun_out/bench_teddy.err
timeout 600 python bench.py --config tsukuba > gpurun_out/bench_tsukuba.json 2> gpurun_out/bench_tsukuba.err
timeout 600 python bench.py --config kitti --steps 500 --warmup 10 > gpurun_out/bench_kitti.json 2> gpurun_out/bench_kitti.err
timeout 900 python bench.py --config mb2014 --steps 20 --warmup 3 > gpurun_out/bench_mb2014.json 2> gpurun_out/bench_mb2014.err
FBS_REF_BUDGET_S=30 timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_teddy.csv python bench.py --steps 20 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_launch.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg -s 2 -c 1 -o gpurun_out/prof_round_agg -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_full.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cost -s 2 -c 1 -o gpurun_out/prof_round_cost -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_cost.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_finalize -s 2 -c 1 -o gpurun_out/prof_round_fin -f python bench.py --steps 3 --warmup 3 --no-extras > /dev/null 2> gpurun_out/ncu_fin.err
ls -la gpurun_out
