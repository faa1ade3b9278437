#!/bin/bash
# timing of prefill kernel variants (tools/exp/libcomet_*.so swapped in), parity-agnostic
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/base.so
for f in tools/exp/libcomet_*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $f"; timeout -s KILL 300 python tools/gemm_sweep.py '[[8192, 57344, 8192, 6], [4096, 11008, 4096, 3]]' 2>&1 | cut -c1-90
done
cp /tmp/base.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
