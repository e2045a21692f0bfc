mkdir -p gpurun_out
./scripts/dev/mma_rate > gpurun_out/mma_rate.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 60 -c 2 -o gpurun_out/gemv_old python scripts/ncu_target.py 4096 4096 1 > gpurun_out/ncu_old.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_gemv --csv --log-file gpurun_out/launches_old.csv python scripts/ncu_target.py 4096 4096 1 > /dev/null 2>&1
cat gpurun_out/mma_rate.txt
