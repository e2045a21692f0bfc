#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_umma -s 6 -c 1 \
  -o gpurun_out/prof_sk python scripts/ncu_target.py 11008 4096 128 > /dev/null 2>&1; echo "prof rc=$?"
