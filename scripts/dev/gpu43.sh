#!/bin/bash
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/dec_launches.csv python scripts/decode_bench.py --layers 4 --gen 3 --reps 1 > gpurun_out/dec43.txt 2>&1; echo rc=$?
