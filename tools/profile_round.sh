#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command + full captures (round 2 layout:
# default bench = LLaMA-3-8B, 4 layers, per-channel weight scales; full captures of the gate_up and down GEMMs)
mkdir -p gpurun_out
# 1) every launch with its device time (cold-cache, serialised)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-group > gpurun_out/launches_bench.json 2>&1; echo launches rc=$?
# 2) full capture of the prefill GEMMs of layers 2 (gate_up) and 3 (down) of the first (eager) step
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:w4ax_gemm_pf -s 2 -c 2 \
  -o gpurun_out/prof_gemm_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-alt-group > /dev/null 2>&1; echo gemm rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:quantize_lane -s 2 -c 2 \
  -o gpurun_out/prof_quant_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-alt-group > /dev/null 2>&1; echo quant rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 2 \
  -o gpurun_out/prof_decode_full python bench.py --config llama3-70b-decode --steps 1 --warmup 3 --no-cpu-baseline --no-alt-group > /dev/null 2>&1; echo decode rc=$?
ls -la gpurun_out/*.ncu-rep
