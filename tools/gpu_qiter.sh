#!/bin/bash
# lane quantizer iteration: parity subset, sweep (fmpq + random perms), one ncu capture
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_quantize_lane.py -m gpu -q -x > gpurun_out/qlane_test.log 2>&1; echo test_rc=$?; tail -2 gpurun_out/qlane_test.log
timeout -s KILL 600 python tools/quant_sweep.py > gpurun_out/quant_sweep.txt 2>&1; echo qs_rc=$?; cat gpurun_out/quant_sweep.txt
timeout -s KILL 600 python tools/quant_sweep.py '[[8192, 4096, 3], [8192, 14336, 11], [16384, 8192, 6], [8192, 28672, 22]]' fmpq > gpurun_out/quant_sweep_fmpq.txt 2>&1; echo qsf_rc=$?; cat gpurun_out/quant_sweep_fmpq.txt
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:quantize_lane -c 1 -o gpurun_out/qprof_fmpq_14336 -f python tools/prof_quant.py 8192 14336 11 fmpq > /dev/null 2>&1; echo ncu_rc=$?
