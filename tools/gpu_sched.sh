#!/bin/bash
# a7 schedule ablation + M sweep (profiles/a7_ablation_r2.txt, profiles/m_sweep_r2.txt)
mkdir -p gpurun_out
timeout -s KILL 900 python tools/a7_ablation.py > gpurun_out/a7_ablation.txt 2>&1; echo abl_rc=$?
timeout -s KILL 1200 python tools/m_sweep.py > gpurun_out/m_sweep.txt 2>&1; echo sweep_rc=$?
