#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:pf_kernel -s 3 -c 1 \
  -o gpurun_out/prof_pf_full python tools/gemm_sweep.py '[[8192, 57344, 8192, 6]]' > gpurun_out/ncu_pf.log 2>&1; echo ncu rc=$?
cp tools/ab/lib_e4.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
timeout -s KILL 600 ncu --set full --clock-control none -k regex:pf_kernel -s 3 -c 1 \
  -o gpurun_out/prof_pf_e4 python tools/gemm_sweep.py '[[8192, 57344, 8192, 6]]' > gpurun_out/ncu_pf2.log 2>&1; echo ncu2 rc=$?
