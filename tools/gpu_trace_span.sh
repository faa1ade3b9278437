#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace_pf(8192, 57344, 8192, 6, cta=0, steps=64)
" > gpurun_out/trace_span.txt 2>&1; echo trace_rc=$?
