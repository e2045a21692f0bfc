#!/bin/bash
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 \
  -o gpurun_out/prof_s8_down python scripts/ncu_target.py 4096 11008 1 > /dev/null 2>&1; echo "prof rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "FAILED|Error|assert|passed|failed" | head -20 > gpurun_out/t33.txt
