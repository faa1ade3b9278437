#!/bin/bash
# raster-group ablation + async host-call test + default bench (e2e)
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/gputest.log
timeout -s KILL 900 python tools/raster_ab.py > gpurun_out/raster_ab.txt 2>&1; echo raster_rc=$?; cat gpurun_out/raster_ab.txt
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_raster.json 2>&1; echo b_rc=$?
tail -1 gpurun_out/bench_raster.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['roofline']['frac'], 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2), d['clocks']['sm_mhz'])"
