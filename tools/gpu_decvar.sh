#!/bin/bash
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/base.so
for f in tools/exp/libcomet_*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $f"; timeout -s KILL 300 python tools/gemm_sweep.py '[[16, 57344, 8192, 6], [16, 8192, 28672, 22], [16, 10240, 8192, 6], [16, 8192, 8192, 6]]' 2>&1 | cut -c1-110
done
cp /tmp/base.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
