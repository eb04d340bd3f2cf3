#!/bin/bash
# One GPU-box script for every session task (run through gpurun from the repo root):
#   tools/gpu.sh smoke                 __graft_entry__.smoke()
#   tools/gpu.sh tests [pytest args]   pytest -m gpu (all tests, -rA)
#   tools/gpu.sh bench CFG [args]      bench.py --config CFG  -> gpurun_out/bench_CFG.json
#   tools/gpu.sh ref                   bench.py --impl reference
#   tools/gpu.sh launches [CFG]        ncu launch list (gpu__time_duration) of a short bench run
#   tools/gpu.sh prof KREGEX TAG [CFG] ncu --set full of one launch of kernels matching KREGEX
#   tools/gpu.sh ab [CFG] [REPS]       interleaved A/B: libfbs.so vs paper_1807_02044_b200/libfbs_exp*.so
# Several tasks chain: tools/gpu.sh smoke tests "bench teddy" launches "prof k_fbs r02"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/gpu_info.txt 2>&1
run_task() {
  set -- $1
  local t=$1; shift
  case $t in
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
    tests)
      timeout 1200 python -m pytest tests -m gpu -q -rA -s "$@" > gpurun_out/gpu_tests.log 2>&1
      echo "tests rc=$?" >> gpurun_out/gpu_tests.log ;;
    bench)
      local c=${1:-teddy}; shift
      timeout 600 python bench.py --config $c "$@" > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
      echo "bench rc=$?" >> gpurun_out/bench_$c.err ;;
    ref)
      FBS_REF_BUDGET_S=30 timeout 600 python bench.py --impl reference --steps 20 --warmup 3 \
        > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err ;;
    launches)
      local c=${1:-teddy}
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 20 --warmup 3 --no-extras \
        > /dev/null 2> gpurun_out/launches_$c.err ;;
    prof)
      local k=$1 tag=$2 c=${3:-teddy}
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
        -o gpurun_out/prof_${tag}_$c -f python bench.py --config $c --steps 3 --warmup 3 --no-extras \
        > /dev/null 2> gpurun_out/prof_${tag}_$c.err ;;
    ab)
      local c=${1:-teddy} reps=${2:-3}
      for i in $(seq 1 $reps); do
        timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras \
          > gpurun_out/ab_default_${c}_$i.json 2>/dev/null
        for v in paper_1807_02044_b200/libfbs_exp*.so; do
          [ -e "$v" ] || continue
          n=$(basename $v .so)
          FBS_LIB=$PWD/$v timeout 300 python bench.py --config $c --steps 1000 --warmup 10 --no-extras \
            > gpurun_out/ab_${n}_${c}_$i.json 2>/dev/null
        done
      done ;;
    *) echo "unknown task $t" >&2 ;;
  esac
}
for task in "$@"; do run_task "$task"; done
ls -la gpurun_out
