#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 -o gpurun_out/prof_s8_big5 python scripts/ncu_target.py 28672 8192 1 > /dev/null 2>&1; echo rc=$?
