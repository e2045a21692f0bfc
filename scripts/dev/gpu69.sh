#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "epi_swiglu or decoder or pre_fused or greedy" > gpurun_out/t69.txt 2>&1
tail -5 gpurun_out/t69.txt
timeout 300 python scripts/dev/decode_parts.py > gpurun_out/parts69.txt 2>&1; tail -2 gpurun_out/parts69.txt
timeout 600 python scripts/decode_bench.py > gpurun_out/dec69.txt 2>&1; tail -2 gpurun_out/dec69.txt
