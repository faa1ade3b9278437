#!/bin/bash
mkdir -p gpurun_out
python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools')
import gemm_sweep as g
g.slow_ctas(16,4096,4096,3); g.slow_ctas(16,57344,8192,6)
"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 3 -c 1 -o gpurun_out/prof_decode70 python tools/gemm_sweep.py '[[16, 57344, 8192, 6]]' > gpurun_out/ncu_dec.log 2>&1; echo ncu rc=$?
