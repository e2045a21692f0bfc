#!/bin/bash
for d in 0 4 8; do for sh in "28672 8192" "11008 4096" "4096 4096"; do
  echo "== dbg $d $sh" >> gpurun_out/tr28.txt
  timeout 120 python scripts/dev/s8_trace.py $sh $d 2>&1 | tail -2 >> gpurun_out/tr28.txt
done; done
timeout 300 python -m pytest tests -m gpu -x -q -k "s8 or linear_vs_oracle or exact or pre_fused" 2>&1 | tail -3 >> gpurun_out/tr28.txt
