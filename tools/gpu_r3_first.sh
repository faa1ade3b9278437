#!/bin/bash
# session start: GPU tests, default bench, quantizer sweep
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_8b.json 2> gpurun_out/bench_8b.err; echo b8_rc=$?
timeout -s KILL 600 python tools/quant_sweep.py > gpurun_out/quant_sweep.txt 2>&1; echo qs_rc=$?
