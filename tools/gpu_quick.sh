#!/bin/bash
# Quick GPU check: parity tests (all, no -x) + the headline bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt
timeout 600 python -m pytest tests -m gpu -q -rA ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_teddy.json 2> gpurun_out/bench_teddy.err
echo "bench rc=$?" >> gpurun_out/bench_teddy.err
