#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
bash tools/gpu_variants2.sh
