#!/bin/bash
# A/B of tools/ab/libcomet_*.so variants (same binding) on one box: bench step + per-kernel times, two rounds
ARGS=${1:-"--steps 20 --warmup 5 --no-cpu-baseline"}
cp paper_2410_12168_b200/libcomet.so /tmp/keep.so
for round in 1 2; do
for f in tools/ab/libcomet_*.so; do
  v=$(basename $f .so); cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  python bench.py $ARGS 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['ms_per_step'],4), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['layer_us']], d['clocks']['sm_mhz'])"
done
done | tee gpurun_out/abv.txt
cp /tmp/keep.so paper_2410_12168_b200/libcomet.so
