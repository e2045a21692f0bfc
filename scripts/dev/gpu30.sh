#!/bin/bash
for v in base s8nowait s8nomath; do
  if [ $v = base ]; then unset TRITRUN_LIB; else export TRITRUN_LIB=$PWD/scripts/dev/var/$v/libtritrun.so; fi
  echo "== $v" >> gpurun_out/ab30.txt
  timeout 300 python scripts/dev/gemv_sweep.py 1 auto 4096x4096,11008x4096,8192x8192,28672x8192 2>&1 | grep -v relerr >> gpurun_out/ab30.txt
  for sh in "28672 8192" "11008 4096"; do timeout 120 python scripts/dev/s8_trace.py $sh 0 2>&1 | tail -1 >> gpurun_out/ab30.txt; done
done
