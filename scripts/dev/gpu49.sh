#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "decoder or greedy" 2>&1 | tail -2 > gpurun_out/t49.txt
timeout 600 python scripts/decode_bench.py >> gpurun_out/t49.txt 2>&1
