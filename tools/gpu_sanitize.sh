#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer_$t.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$t.txt
done
