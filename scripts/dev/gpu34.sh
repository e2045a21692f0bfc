#!/bin/bash
timeout 300 python scripts/dev/gemv_sweep.py 1,2 auto 4096x4096,11008x4096,4096x11008,8192x8192,28672x8192 2>&1 | grep -v relerr > gpurun_out/sw34.txt
for sh in "28672 8192" "11008 4096" "4096 11008"; do timeout 120 python scripts/dev/s8_trace.py $sh 0 2>&1 | tail -1 >> gpurun_out/sw34.txt; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 \
  -o gpurun_out/prof_s8_down2 python scripts/ncu_target.py 4096 11008 1 > /dev/null 2>&1; echo "prof rc=$?"
