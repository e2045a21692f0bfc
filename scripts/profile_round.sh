#!/bin/bash
# GPU-side evidence for a round: bench JSON, ncu launch list of the bench command, and one
# full ncu capture of each hot kernel.  Run: gpurun --timeout 2400 -- bash scripts/profile_round.sh
set -u
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gemv|k_gemm" -c 300 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --sweep "" --extras "" --cpu-seconds 0.1 > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 6 -c 1 \
  -o gpurun_out/prof_gemv env COSCHED=1 python scripts/ncu_target.py 11008 4096 1 > /dev/null 2>&1; echo "gemv prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_umma -s 6 -c 1 \
  -o gpurun_out/prof_umma python scripts/ncu_target.py 11008 4096 128 > /dev/null 2>&1; echo "umma prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_umma -s 6 -c 1 \
  -o gpurun_out/prof_u16 python scripts/ncu_target.py 11008 4096 16 > /dev/null 2>&1; echo "umma b16 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv_s8 -s 6 -c 1 \
  -o gpurun_out/prof_q1 env FMT=TQ1 python scripts/ncu_target.py 8192 8192 1 > /dev/null 2>&1; echo "q1 prof rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv_chain -s 2 -c 1 \
  -o gpurun_out/prof_chain python scripts/dev/ncu_chain.py 8 > /dev/null 2>&1; echo "chain prof rc=$?"
