mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 40 -c 1 -o gpurun_out/gemv_new_big python scripts/ncu_target.py 28672 8192 1 > gpurun_out/ncu4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 40 -c 1 -o gpurun_out/gemv_new_4k python scripts/ncu_target.py 4096 4096 1 >> gpurun_out/ncu4.log 2>&1
tail -3 gpurun_out/ncu4.log
