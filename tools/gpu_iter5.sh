#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_fmpq_aux.py -m gpu -q > gpurun_out/gputest_aux.log 2>&1; echo test_rc=$?; tail -3 gpurun_out/gputest_aux.log
timeout -s KILL 600 python tools/aux_bench.py > gpurun_out/aux_bench.txt 2>&1; echo aux_rc=$?; cat gpurun_out/aux_bench.txt
