#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/t52.txt
bash scripts/profile_round.sh >> gpurun_out/t52.txt 2>&1
