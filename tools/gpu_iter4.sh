#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -3 gpurun_out/gputest.log
timeout -s KILL 300 python tools/gemm_sweep.py '[[8192, 57344, 8192, 6], [8192, 4096, 4096, 3], [8192, 4096, 14336, 11], [4096, 11008, 4096, 3], [4096, 4096, 4096, 3], [512, 4096, 4096, 3]]' > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt | cut -c1-100
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench8b.json 2> gpurun_out/bench8b.err; echo b8_rc=$?; tail -2 gpurun_out/bench8b.err
