#!/bin/bash
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/base.so
for f in /tmp/base.so tools/exp/libcomet_*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $f"; timeout -s KILL 300 python tools/quant_sweep.py '[[8192, 8192, 6], [8192, 28672, 22]]' 2>&1 | cut -c1-100
done
cp /tmp/base.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
