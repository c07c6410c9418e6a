#!/bin/bash
# A/B timing of an environment switch on the default bench (same box, interleaved)
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in "" "$AB_ENV"; do
    r=$(env $v timeout 300 python bench.py --no-cpu-baseline --steps 8 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["tick_kernel_ms"])')
    echo "[${v:-base}] $r" >> gpurun_out/ab.txt
  done
done
