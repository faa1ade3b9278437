#!/bin/bash
# prefill TMA-store epilogue check: full GPU suite, per-K sweep, default bench
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo test_rc=$?; tail -3 gpurun_out/gputest.log
timeout -s KILL 600 python tools/gemm_sweep.py '[[8192, 28672, 4096, 3], [8192, 28672, 8192, 6], [8192, 28672, 2048, 2], [8192, 57344, 8192, 6], [8192, 4096, 14336, 11], [4096, 11008, 4096, 3]]' > gpurun_out/kdep2.txt 2>&1; echo kdep_rc=$?; cut -c1-120 gpurun_out/kdep2.txt
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('8b', round(d['value'],1), [round(x,1) for x in d['gemm_us']], [round(x,1) for x in d['quantize_us']], d['roofline']['frac'], d['clocks']['sm_mhz'])"
