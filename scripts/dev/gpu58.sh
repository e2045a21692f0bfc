#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 10 -c 1 -o gpurun_out/prof_pre2 python scripts/dev/ncu_pre.py 3072 9216 2 > /dev/null 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 10 -c 1 -o gpurun_out/prof_pre0 python scripts/ncu_target.py 3072 9216 1 > /dev/null 2>&1; echo rc=$?
