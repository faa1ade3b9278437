#!/bin/bash
# A/B of the prefill kernels (TMEM-A pf vs SMEM-operand 2sm) + parity of the default path
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/smoke.log
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/parity.log 2>&1; echo parity_rc=$?; tail -15 gpurun_out/parity.log
for impl in pf 2sm; do
  for cfg in llama2-7b llama3-70b; do
    COMET_PREFILL=$impl timeout -s KILL 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${impl}_${cfg}.json 2> gpurun_out/ab_${impl}_${cfg}.err; echo "$impl $cfg rc=$?"
    python -c "import json;d=json.load(open('gpurun_out/ab_${impl}_${cfg}.json'));print('  ', round(d['value'],1), d['unit'], 'gemm_us', [round(x,1) for x in d['gemm_us']], 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -3 gpurun_out/ab_${impl}_${cfg}.err
  done
done
