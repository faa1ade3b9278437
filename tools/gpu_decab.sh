#!/bin/bash
# decode A/B over tools/ab variants: parity subset + M sweep of the decode shapes
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "decode or split or c1 or full or power" > /tmp/t.log 2>&1; echo "$(basename $f) test_rc=$?"; tail -1 /tmp/t.log
done
for round in 1 2; do
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $(basename $f)"
  timeout -s KILL 300 python tools/gemm_sweep.py '[[16, 57344, 8192, 6], [16, 8192, 28672, 22], [1, 57344, 8192, 6], [32, 57344, 8192, 6], [64, 57344, 8192, 6], [128, 57344, 8192, 6], [16, 28672, 4096, 3], [16, 4096, 14336, 11]]' 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(d['M'], d['N'], d['K'], round(d['us'], 1), round(d['GBs']))
    except Exception: print(l.strip()[:200])
"
done
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so
