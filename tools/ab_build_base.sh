#!/bin/bash
# build libcomet from a git revision (default HEAD) into tools/ab/libcomet_base.so for tools/gpu_ab.sh
REV=${1:-HEAD}
rm -rf /tmp/ab_src && mkdir -p /tmp/ab_src tools/ab
git archive "$REV" paper_2410_12168_b200/csrc include | tar -x -C /tmp/ab_src
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -I /tmp/ab_src/include -o tools/ab/libcomet_base.so /tmp/ab_src/paper_2410_12168_b200/csrc/comet_api.cu
