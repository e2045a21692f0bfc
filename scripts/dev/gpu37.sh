#!/bin/bash
for d in 0 1; do for sh in "11008 4096" "4096 11008" "28672 8192"; do
  echo "== dbg $d $sh" >> gpurun_out/tr37.txt
  timeout 120 python scripts/dev/s8_trace.py $sh $d 2>&1 | tail -1 >> gpurun_out/tr37.txt
done; done
timeout 300 python scripts/dev/gemv_sweep.py 1,2 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr >> gpurun_out/tr37.txt
