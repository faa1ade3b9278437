#!/bin/bash
# one full ncu capture of the decode GEMM (llama3-70b gate_up, M=16) with source counters
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 \
  -o gpurun_out/dec_full python tools/gemm_sweep.py '[[16, 57344, 8192, 6]]' > gpurun_out/dec_full.log 2>&1; echo decode rc=$?
ls -la gpurun_out/*.ncu-rep
