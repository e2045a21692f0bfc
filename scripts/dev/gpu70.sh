#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/dev/epi_agree.py > gpurun_out/agree70.txt 2>&1; tail -3 gpurun_out/agree70.txt
