#!/bin/bash
mkdir -p gpurun_out
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace(16, 57344, 8192, 6, cta=0, units=24)
g.roles(16, 57344, 8192, 6, cta=0)
g.cta_times(16, 57344, 8192, 6)
g.trace(16, 8192, 28672, 22, cta=0, units=24)
g.cta_times(16, 8192, 28672, 22)
" > gpurun_out/dec_trace.txt 2>&1; echo rc=$?
cat gpurun_out/dec_trace.txt
