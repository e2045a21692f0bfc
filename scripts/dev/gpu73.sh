#!/bin/bash
mkdir -p gpurun_out
for shp in "11008 4096 128" "4096 4096 128" "4096 11008 128" "11008 4096 16" "4096 4096 16"; do
  timeout 120 python scripts/dev/umma_probe.py $shp 0,1,2,3 0,1,2 >> gpurun_out/p73.txt 2>&1
done
cat gpurun_out/p73.txt
