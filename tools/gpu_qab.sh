#!/bin/bash
# quantizer A/B: parity subset on the tree's library, then sweep + bench per tools/ab variant
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "quantize or bf16 or static or extremes or c1_tiny or ragged or linear or prefill" > gpurun_out/q2test.log 2>&1; echo qtest_rc=$?; tail -3 gpurun_out/q2test.log
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
for round in 1 2; do
for f in tools/ab/lib*.so; do
  cp $f paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $(basename $f)"
  timeout -s KILL 120 python tools/quant_sweep.py '[[8192, 4096, 3], [8192, 14336, 11]]' 2>&1 | cut -c1-100
  timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $f)', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['clocks']['sm_mhz'])"
done
done
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so
