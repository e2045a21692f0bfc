#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "s8 or linear_vs_oracle or exact or pre_fused or uniform or partition or decoder" 2>&1 | tail -2 > gpurun_out/t50.txt
timeout 300 python scripts/dev/gemv_sweep.py 1,2 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr >> gpurun_out/t50.txt
for sh in "11008 4096" "4096 11008"; do timeout 120 python scripts/dev/s8_trace.py $sh 0 2>&1 | tail -1 >> gpurun_out/t50.txt; done
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'])" >> gpurun_out/t50.txt
