#!/bin/bash
mkdir -p gpurun_out
bash tools/gpu_test_pf_ab.sh 2>/dev/null
cp paper_2410_12168_b200/libcomet.so /tmp/tree.so
cp tools/ab/lib2_pfirst.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or full or power or ragged or linear" > gpurun_out/pfirst_test.log 2>&1; echo pfirst_test_rc=$?; tail -1 gpurun_out/pfirst_test.log
cp /tmp/tree.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
bash tools/gpu_pfab.sh
bash tools/gpu_trace_span.sh
