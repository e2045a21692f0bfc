#!/bin/bash
timeout 600 python -m pytest tests -m gpu -x -q -k "umma or tq1 or decoder or baseline_shapes or matches_gemv" 2>&1 | tail -1 > gpurun_out/t65.txt
timeout 300 python scripts/dev/gemv_sweep.py 16,64,128 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr >> gpurun_out/t65.txt
