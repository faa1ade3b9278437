#!/bin/bash
mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace2(4096, 4096, 4096, 3, cta=0, steps=48)" > gpurun_out/trace2.txt 2>&1
