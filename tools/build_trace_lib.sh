#!/bin/bash
# libcomet with per-role cycle counters and per-step event traces compiled in
# (-DCOMET_TRACE) -> tools/trace/libcomet_trace.so. Use via tools/with_trace_lib.sh.
mkdir -p tools/trace
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -I include -DCOMET_TRACE $TRACE_FLAGS -o tools/trace/libcomet_trace.so paper_2410_12168_b200/csrc/comet_api.cu
