#!/bin/bash
# one full ncu capture of the prefill GEMM (7B layer1 shape) with source-level sampling
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:pf_kernel -s 3 -c 1 \
  -o gpurun_out/prof_pf python tools/gemm_sweep.py '[[4096, 11008, 4096, 3]]' > gpurun_out/ncu_pf.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_pf.log
