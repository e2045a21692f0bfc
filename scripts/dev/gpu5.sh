mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 5 -c 1 -o gpurun_out/prof_$1 python scripts/ncu_target.py $2 $3 $4 > gpurun_out/ncu_$1.log 2>&1; tail -2 gpurun_out/ncu_$1.log
