#!/bin/bash
# smoke + GPU parity, then A/B bench of libfbs.so vs paper_1807_02044_b200/libfbs_exp*.so
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
bash tools/gpu_ab.sh
