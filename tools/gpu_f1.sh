#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_allgather_fused.py -m gpu -q -x > gpurun_out/f1_test.log 2>&1; echo f1_rc=$?; tail -15 gpurun_out/f1_test.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python bench.py --no-cpu-baseline > gpurun_out/bench_8b.json 2> gpurun_out/bench_8b.err; echo b8_rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_8b.json')); print(d['value'], d['ms_per_step'], 'q', [round(x,1) for x in d['quantize_us']], 'layer', [round(x,1) for x in d['layer_us']], 'gemm', [round(x,1) for x in d['gemm_us']], d['roofline']['frac'])"
