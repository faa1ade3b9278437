#!/bin/bash
# one iteration: GPU tests, GEMM sweep (70B gate_up / 7B), per-block trace, 8B bench
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -4 gpurun_out/gputest.log
timeout -s KILL 300 python tools/gemm_sweep.py '[[8192, 57344, 8192, 6], [8192, 8192, 28672, 22], [4096, 11008, 4096, 3]]' > gpurun_out/sweep.txt 2>&1; cat gpurun_out/sweep.txt
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace_pf(8192, 57344, 8192, 6, cta=0, steps=64)
" > gpurun_out/trace_pf.txt 2>&1; echo trace_rc=$?; tail -1 gpurun_out/trace_pf.txt
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench8b.json 2> gpurun_out/bench8b.err; echo b8_rc=$?
