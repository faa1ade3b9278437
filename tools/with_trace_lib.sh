#!/bin/bash
# run a command with the COMET_TRACE library swapped in (GPU box), then restore
cp paper_2410_12168_b200/libcomet.so /tmp/tree_lib.so
cp tools/trace/libcomet_trace.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
"$@"; rc=$?
cp /tmp/tree_lib.so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
exit $rc
