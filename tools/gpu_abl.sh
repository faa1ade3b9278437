#!/bin/bash
# bench A/B over tools/ab variants printing the step, layer (linear) and GEMM times
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for round in 1 2; do
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt-group $1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $f)', round(d['value'],1), 'layer', [round(x,1) for x in d['layer_us']], 'gemm', [round(x,1) for x in d['gemm_us']], 'e2e', round(d['e2e']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so
