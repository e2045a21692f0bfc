#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t71.txt 2>&1
tail -5 gpurun_out/t71.txt
