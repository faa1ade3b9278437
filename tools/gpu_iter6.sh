#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "linear" > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python bench.py --no-cpu-baseline --no-alt-group > gpurun_out/bench8b.json 2> gpurun_out/bench8b.err; echo b8_rc=$?; tail -2 gpurun_out/bench8b.err
