#!/bin/bash
# A/B timing of an environment switch (same box, interleaved).
# AB_ENV="VAR=1" [WORKLOADS="config3 config5"] [STEPS=8] bash tools/ab.sh
mkdir -p gpurun_out
for w in ${WORKLOADS:-config3}; do
  for i in 1 2 3; do
    for v in "" "$AB_ENV"; do
      r=$(env $v timeout 300 python bench.py --workload $w --no-cpu-baseline --steps ${STEPS:-8} 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["tick_kernel_ms"])')
      echo "$w [${v:-base}] $r" >> gpurun_out/ab.txt
    done
  done
done
