#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "s8 or linear_vs_oracle or exact or pre_fused or uniform or partition or decoder or baseline" 2>&1 | tail -3 > gpurun_out/t51.txt
timeout 300 python scripts/dev/gemv_sweep.py 1,2,3,4 auto,gemv_f16 4096x4096,11008x4096,4096x11008,8192x8192 2>&1 | grep -v relerr >> gpurun_out/t51.txt
