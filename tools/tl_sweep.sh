#!/bin/bash
# timeline of the TC kernel under debug flags (timing experiments only)
mkdir -p gpurun_out
for f in ${FLAGS:-0 32}; do
  echo "=== RANC_DEBUG_FLAGS=$f" >> gpurun_out/tl_sweep.txt
  RANC_DEBUG_FLAGS=$f python tools/timeline.py 2>&1 | grep -A12 "t=2" >> gpurun_out/tl_sweep.txt
done
