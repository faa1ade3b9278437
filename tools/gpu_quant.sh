#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 300 python tools/quant_sweep.py > gpurun_out/quant_sweep.txt 2>&1; echo rc=$?; cat gpurun_out/quant_sweep.txt
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quantize -s 5 -c 1 -o gpurun_out/prof_quant python tools/quant_sweep.py '[[4096, 4096, 3]]' > /dev/null 2>&1; echo ncu rc=$?
