#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "linear or c1_tiny or ragged or power" > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench8b.json 2> gpurun_out/bench8b.err; echo b8_rc=$?; tail -2 gpurun_out/bench8b.err
timeout -s KILL 1200 python tools/c5_sweep.py 16,8192 K > gpurun_out/c5_sweep.txt 2>&1; echo c5_rc=$?
