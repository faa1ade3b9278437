#!/bin/bash
# time every tools/ab/var_*.so with the same bench args (the library is swapped in place)
# usage: bash tools/gpu_variants.sh "<bench args>" ["<bench args 2>" ...]
mkdir -p gpurun_out
cp paper_2410_12168_b200/libcomet.so /tmp/keep.so
for ARGS in "$@"; do
  echo "== $ARGS"
  for so in tools/ab/var_*.so; do
    cp $so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
    timeout -s KILL 300 python bench.py $ARGS 2>/tmp/err.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $so)', round(d['value'],1), d['unit'], [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -2 /tmp/err.txt
  done
done
cp /tmp/keep.so paper_2410_12168_b200/libcomet.so
