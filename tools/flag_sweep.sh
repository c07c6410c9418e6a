#!/bin/bash
# bench under RANC_DEBUG_FLAGS variants (timing experiments only)
mkdir -p gpurun_out
for f in ${FLAGS:-0 1 2 3}; do
  echo "=== RANC_DEBUG_FLAGS=$f $(RANC_DEBUG_FLAGS=$f timeout 300 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["tick_kernel_ms"])')" >> gpurun_out/flag_sweep.txt
done
