#!/bin/bash
mkdir -p gpurun_out
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace3(8192, 57344, 8192, 6, cta=2, steps=30)
g.trace3(8192, 57344, 8192, 6, cta=0, steps=30)
" > gpurun_out/trace3.txt 2>&1; echo rc=$?
cat gpurun_out/trace3.txt | head -140
