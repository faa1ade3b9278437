#!/bin/bash
# trace3 of the 70B gate_up shape with the default trace lib and tools/trace/alt/*.so
mkdir -p gpurun_out
for lib in tools/trace/libcomet_trace.so tools/trace/alt/*.so; do
  echo "=== $lib"
  cp $lib /tmp/cur_trace.so
  cp paper_2410_12168_b200/libcomet.so /tmp/tree_lib.so
  cp /tmp/cur_trace.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  python -c "
import sys; sys.path.insert(0, 'tools'); import gemm_sweep as g
g.trace3(8192, 57344, 8192, 6, cta=2, steps=14)
" 2>&1 | tail -22
  cp /tmp/tree_lib.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
done
