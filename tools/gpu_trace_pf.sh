#!/bin/bash
# per-block event trace of the prefill kernel (COMET_TRACE build, built here: tools/build_trace_lib.sh)
mkdir -p gpurun_out
bash tools/with_trace_lib.sh python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace_pf(8192, 57344, 8192, 6, cta=0, steps=64)
g.trace_pf(8192, 57344, 8192, 6, cta=0, steps=64, group='128')
" > gpurun_out/trace_pf.txt 2>&1; echo trace_rc=$?
timeout -s KILL 900 python bench.py --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench8b.json 2> gpurun_out/bench8b.err; echo b8_rc=$?
tail -3 gpurun_out/bench8b.err
