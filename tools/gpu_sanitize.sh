#!/bin/bash
# compute-sanitizer over every GEMM path (memcheck / racecheck / synccheck)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.txt
done
