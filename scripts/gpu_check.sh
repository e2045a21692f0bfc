#!/bin/bash
# One gpurun call: GPU parity tests, smoke, a short bench, and the ncu launch list.
# Usage (from this container): gpurun --timeout 1500 -- bash scripts/gpu_check.sh [tests|bench|ncu|all]
set -u
mkdir -p gpurun_out
what=${1:-all}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == all || $what == tests ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
fi
if [[ $what == all || $what == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --cpu-seconds 0.1 > gpurun_out/ncu_bench.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
fi
tail -3 gpurun_out/*.log
