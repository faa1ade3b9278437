#!/bin/bash
# run the bench against every tools/ab/lib*.so variant (2 rounds), restoring the tree's library
ARGS=${1:-"--steps 10 --warmup 3 --no-cpu-baseline"}
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for round in 1 2; do
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  python bench.py $ARGS 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $f)', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['clocks']['sm_mhz'])"
done
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so
