#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/t44.txt
timeout 300 python scripts/dev/gemv_sweep.py 1 auto 4096x4096,11008x4096,4096x11008,3072x3072,3072x9216 2>&1 | grep -v relerr >> gpurun_out/t44.txt
timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/t44.txt
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'])" >> gpurun_out/t44.txt
