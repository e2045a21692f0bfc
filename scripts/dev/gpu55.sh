#!/bin/bash
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'], d['e2e']['value'])" > gpurun_out/t55.txt
timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/t55.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "s8 or linear_vs_oracle or pre_fused or decoder or chain" 2>&1 | tail -1 >> gpurun_out/t55.txt
