#!/bin/bash
mkdir -p gpurun_out
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace_pf(8192, 28672, 4096, 3, cta=0, steps=64, group='K')
" > gpurun_out/trace_pf8b.txt 2>&1; echo rc=$?
