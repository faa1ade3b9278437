#!/bin/bash
# parity + prefill bench (per-channel and group-128) + the 70B prefill config
mkdir -p gpurun_out
bash tools/gpu_test.sh
for g in channel 128; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --group $g 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefill group=$g', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], round(d['roofline']['frac'],3), d['clocks'])"
done
