#!/bin/bash
# round-2 first call: microbenchmarks (pipe rates, fp8 MMA exactness/rate), GPU tests, baseline bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout -s KILL 120 ./tools/mb_fp8 > gpurun_out/mb_fp8.txt 2>&1; echo mb_fp8_rc=$?
timeout -s KILL 120 ./tools/microbench > gpurun_out/mb.txt 2>&1; echo mb_rc=$?
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -3 gpurun_out/gputest.log
timeout -s KILL 600 python bench.py --config llama3-70b --no-cpu-baseline > gpurun_out/bench70.json 2> gpurun_out/bench70.err; echo b70_rc=$?
timeout -s KILL 600 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo b7_rc=$?
