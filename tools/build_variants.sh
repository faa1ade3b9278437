#!/bin/bash
# build libcomet variants with -D flags into tools/ab/libcomet_<name>.so
# usage: bash tools/build_variants.sh name1 "-DFOO=1 -DBAR=2" name2 "..."
mkdir -p tools/ab
while [ $# -ge 2 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr -I include $2 -o tools/ab/libcomet_$1.so paper_2410_12168_b200/csrc/comet_api.cu &
  shift 2
done
wait
