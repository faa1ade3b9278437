#!/bin/bash
# prefill epilogue A/B over tools/ab variants: per-K sweep
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for round in 1 2; do
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $(basename $f)"
  timeout -s KILL 300 python tools/gemm_sweep.py '[[8192, 28672, 4096, 3], [8192, 28672, 8192, 6], [8192, 28672, 2048, 2], [8192, 57344, 8192, 6], [8192, 4096, 14336, 11]]' 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l); print(d['M'], d['N'], d['K'], round(d['us'], 1), round(d['TOPS']))
    except Exception: print(l.strip()[:200])
"
done
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so
