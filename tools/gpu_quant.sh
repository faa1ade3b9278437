#!/bin/bash
# quantizer: parity (bit-exact planes) + bandwidth sweep
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -k "quantize or bf16 or static or extremes or c1_tiny or ragged" > gpurun_out/qtest.log 2>&1; echo qtest_rc=$?; tail -3 gpurun_out/qtest.log
timeout -s KILL 300 python tools/quant_sweep.py > gpurun_out/quant_sweep.txt 2>&1; cat gpurun_out/quant_sweep.txt
