#!/bin/bash
for d in 0 4 8; do for sh in "28672 8192" "11008 4096" "4096 11008"; do
  echo "== dbg $d $sh" >> gpurun_out/tr32.txt
  timeout 120 python scripts/dev/s8_trace.py $sh $d 2>&1 | tail -1 >> gpurun_out/tr32.txt
done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/tr32.txt
