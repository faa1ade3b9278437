#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "linear or quantize" > gpurun_out/p16test.log 2>&1; echo test_rc=$?; tail -1 gpurun_out/p16test.log
for i in 1 2; do
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt-group 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['roofline']['frac'], 'e2e', round(d['e2e']['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
