#!/bin/bash
# per-block cost vs K (tile length) for the prefill kernel + 8B gate_up trace across a tile boundary
mkdir -p gpurun_out
timeout -s KILL 600 python tools/gemm_sweep.py '[[8192, 28672, 4096, 3], [8192, 28672, 8192, 6], [8192, 28672, 16384, 12], [8192, 57344, 4096, 3], [8192, 57344, 8192, 6], [8192, 28672, 2048, 2], [8192, 28672, 1024, 1]]' > gpurun_out/kdep.txt 2>&1; echo kdep_rc=$?
timeout -s KILL 600 bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace_pf(8192, 28672, 4096, 3, cta=0, steps=64)
" > gpurun_out/trace_pf8b.txt 2>&1; echo trace_rc=$?
