#!/bin/bash
# quick GPU check: smoke + parity (optionally a -k filter as $1)
mkdir -p gpurun_out
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${1:+-k "$1"} > gpurun_out/parity.log 2>&1; echo parity_rc=$?; tail -25 gpurun_out/parity.log
