#!/bin/bash
timeout 300 python scripts/dev/gemv_sweep.py 1,2,4,8 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr > gpurun_out/sw31.txt
for sh in "28672 8192" "11008 4096"; do timeout 120 python scripts/dev/s8_trace.py $sh 0 2>&1 | tail -1 >> gpurun_out/sw31.txt; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 >> gpurun_out/sw31.txt
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'], d['e2e'])" >> gpurun_out/sw31.txt
