#!/bin/bash
timeout 300 python scripts/dev/gemv_sweep.py 1 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr > gpurun_out/t63.txt
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'])" >> gpurun_out/t63.txt
timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/t63.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "s8 or linear_vs_oracle or pre_fused or decoder or cosched" 2>&1 | tail -1 >> gpurun_out/t63.txt
