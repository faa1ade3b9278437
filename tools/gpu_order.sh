#!/bin/bash
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for f in tools/ab/lib2_order2.so tools/ab/lib3_order3.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or full or power" > /tmp/t.log 2>&1; echo "$(basename $f) test_rc=$?"; tail -1 /tmp/t.log
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
bash tools/gpu_pfab.sh
