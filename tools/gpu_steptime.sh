#!/bin/bash
cp paper_2410_12168_b200/libcomet.so /tmp/keep.so
for so in tools/ab/var_*.so; do
  cp $so paper_2410_12168_b200/libcomet.so; touch paper_2410_12168_b200/libcomet.so
  echo "== $(basename $so)"; timeout 300 python tools/step_time.py "$@" 2>&1 | grep step_us
done
cp /tmp/keep.so paper_2410_12168_b200/libcomet.so
