#!/bin/bash
# Round-2 record session: both paths, all configs, reference arm, ncu launch lists and
# full captures of the dominant kernel of each path at the headline config.
mkdir -p gpurun_out/r02
o=gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/gpu_info.txt
for p in volume fused; do
  timeout 600 python bench.py --path $p > $o/bench_teddy_$p.json 2> $o/bench_teddy_$p.err
  timeout 600 python bench.py --path $p --no-graph --steps 1000 --warmup 10 --no-extras > $o/bench_teddy_${p}_eager.json 2>/dev/null
  timeout 600 python bench.py --path $p --config tsukuba --steps 1000 --warmup 10 > $o/bench_tsukuba_$p.json 2> $o/bench_tsukuba_$p.err
  timeout 600 python bench.py --path $p --config kitti --steps 300 --warmup 10 > $o/bench_kitti_$p.json 2> $o/bench_kitti_$p.err
  timeout 900 python bench.py --path $p --config mb2014 --steps 10 --warmup 3 > $o/bench_mb2014_$p.json 2> $o/bench_mb2014_$p.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_teddy_$p.csv \
    python bench.py --path $p --steps 20 --warmup 3 --no-extras --no-graph > /dev/null 2>&1
done
FBS_REF_BUDGET_S=30 timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_agg -s 2 -c 1 -o $o/prof_agg_teddy -f \
  python bench.py --path volume --steps 3 --warmup 3 --no-extras --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cost -s 2 -c 1 -o $o/prof_cost_teddy -f \
  python bench.py --path volume --steps 3 --warmup 3 --no-extras --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fbs_ws -s 2 -c 1 -o $o/prof_fbsws_teddy -f \
  python bench.py --path fused --steps 3 --warmup 3 --no-extras --no-graph > /dev/null 2>&1
# summarise the captures here (the .ncu-rep files are too large to bring back)
mkdir -p gpurun_out/r02_summary
cp profiles/ncu_summary.json gpurun_out/r02_summary/ 2>/dev/null
python tools/make_profiles.py r02 $o --out gpurun_out/r02_summary > gpurun_out/r02_summary/make_profiles.log 2>&1
mkdir -p /tmp/ncu_reps && mv $o/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
ls -la $o gpurun_out/r02_summary
