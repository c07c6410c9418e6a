#!/bin/bash
# One JSON line per workload (N=1), both kernels where the tensor-core path applies.
mkdir -p gpurun_out
out=gpurun_out/bench_all.jsonl
: > $out
for w in config3 config2 config1 vmm32 vmm256 vmm1024 config5 config5g config5z stream sweep8 config3w bigcore; do
  for k in auto popc; do
    timeout 600 python bench.py --workload $w --kernel $k --steps ${STEPS:-5} --warmup 3 ${EXTRA} 2>>gpurun_out/bench_all.err | tail -1 >> $out
  done
done
