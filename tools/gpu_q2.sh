#!/bin/bash
# quantizer change check: parity subset, bandwidth sweep, default bench
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "quantize or bf16 or static or extremes or c1_tiny or ragged or linear or prefill" > gpurun_out/q2test.log 2>&1; echo qtest_rc=$?; tail -3 gpurun_out/q2test.log
timeout -s KILL 300 python tools/quant_sweep.py > gpurun_out/quant_sweep.txt 2>&1; cat gpurun_out/quant_sweep.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d.get('layer_us'), d['clocks']['sm_mhz'])"
