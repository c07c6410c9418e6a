#!/bin/bash
# One GPU session: smoke, GPU tests, int peaks, bench, ncu launch list + full capture.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/int_peaks tools/int_peaks.cu && timeout 120 /tmp/int_peaks > gpurun_out/int_peaks.json 2>&1; echo "peaks rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --kernel popc --no-cpu-baseline > gpurun_out/bench_popc.log 2>&1; echo "bench-popc rc=$?" >> gpurun_out/status.txt
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu-launch rc=$?" >> gpurun_out/status.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick_ -s 40 -c 1 -o gpurun_out/prof -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> gpurun_out/status.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tick_ -s 40 -c 1 -o gpurun_out/prof_popc -f python bench.py --kernel popc --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_popc.log 2>&1; echo "ncu-full-popc rc=$?" >> gpurun_out/status.txt
fi
