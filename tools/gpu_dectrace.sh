#!/bin/bash
mkdir -p gpurun_out
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.slowest_roles(16, 8192, 28672, 22)
g.trace(16, 8192, 28672, 22, cta=5, units=30)
g.slowest_roles(16, 57344, 8192, 6)
g.trace(16, 57344, 8192, 6, cta=5, units=30)
" > gpurun_out/dectrace.txt 2>&1; echo rc=$?
