#!/bin/bash
# parity of one variant library: bash tools/gpu_var_parity.sh tools/ab/var_X.so [pytest -k expr]
cp paper_2410_12168_b200/libcomet.so /tmp/keep_p.so
cp $1 paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu ${2:+-k "$2"} 2>&1 | tail -5
cp /tmp/keep_p.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
