#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "decoder or greedy or attn" 2>&1 | tail -3 > gpurun_out/t47.txt
timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/t47.txt
timeout 600 python scripts/decode_bench.py >> gpurun_out/t47.txt 2>&1
