#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "pre_fused or decoder or greedy" 2>&1 | tail -1 > gpurun_out/t59.txt
timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/t59.txt
timeout 600 python scripts/decode_bench.py >> gpurun_out/t59.txt 2>&1
