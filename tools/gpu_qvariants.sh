#!/bin/bash
# run the fmpq quantizer sweep for each tools/ab/libcomet_*.so variant (swapped in as libcomet.so)
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/keep.so
for f in tools/ab/libcomet_*.so; do
  v=$(basename $f .so); cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $v"; timeout -s KILL 300 python tools/quant_sweep.py "${1:-[[8192, 4096, 3], [8192, 14336, 11], [8192, 28672, 22]]}" fmpq 2>&1 | grep fmpq
done | tee gpurun_out/qvariants.txt
cp /tmp/keep.so paper_2410_12168_b200/libcomet.so
