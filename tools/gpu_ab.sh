#!/bin/bash
# A/B: tools/ab/libcomet_base.so vs the working tree's libcomet.so on the same box
# usage: bash tools/gpu_ab.sh "<bench args>"
ARGS=${1:-"--steps 10 --warmup 3 --no-cpu-baseline"}
cp paper_2410_12168_b200/libcomet.so /tmp/new.so
for round in 1 2; do
for v in base new; do
  if [ $v = base ]; then cp tools/ab/libcomet_base.so paper_2410_12168_b200/libcomet.so; else cp /tmp/new.so paper_2410_12168_b200/libcomet.so; fi
  touch paper_2410_12168_b200/libcomet.so
  python bench.py $ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['clocks']['sm_mhz'])"
done
done
cp /tmp/new.so paper_2410_12168_b200/libcomet.so
