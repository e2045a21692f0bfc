#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/dev/gemv_sweep.py 1,4,8 auto 8192x8192,28672x8192,8192x28672,11008x4096 > gpurun_out/sweep22.txt 2>&1; echo "sweep rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 \
  -o gpurun_out/prof_gemv_big python scripts/ncu_target.py 28672 8192 1 > /dev/null 2>&1; echo "prof rc=$?"
