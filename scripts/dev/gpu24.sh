#!/bin/bash
mkdir -p gpurun_out
for v in nowait; do
  export TRITRUN_LIB=$PWD/scripts/dev/var/$v/libtritrun.so
  echo "== $v" >> gpurun_out/ab24.txt
  timeout 300 python scripts/dev/gemv_sweep.py 1 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr >> gpurun_out/ab24.txt
done
