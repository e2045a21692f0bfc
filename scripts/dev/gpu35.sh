#!/bin/bash
for d in 0 4 12; do for sh in "11008 4096" "4096 11008"; do
  echo "== dbg $d $sh" >> gpurun_out/tr35.txt
  timeout 120 python scripts/dev/s8_trace.py $sh $d 2>&1 | tail -1 >> gpurun_out/tr35.txt
done; done
