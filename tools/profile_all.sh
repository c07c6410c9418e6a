#!/bin/bash
# One ncu --set full capture of the dominant tick kernel of every bench
# workload (run on the GPU box from the repo root):
#   bash tools/profile_all.sh [tag] [workload ...]
# -> gpurun_out/prof_<tag>_<workload>.ncu-rep, summarised here with
#    python tools/ncu_summary.py counters gpurun_out/prof_<tag>_*.ncu-rep
tag=${1:-r02}; shift
wls=${@:-config3 config3_popc config2 config1 vmm32 vmm256 vmm1024 config5 config5g stream}
mkdir -p gpurun_out
for w in $wls; do
  args="--workload $w"; skip=40
  case $w in
    config3_popc) args="--workload config3 --kernel popc";;
    config2|vmm32|vmm256|config1|stream) skip=2;;       # one cooperative launch per step
    vmm1024) skip=200;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick_ -s $skip -c 1 \
    -o gpurun_out/prof_${tag}_$w -f python bench.py $args --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/prof_${tag}_$w.log 2>&1
  echo "$w rc=$?"
done
