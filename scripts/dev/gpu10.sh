timeout 600 python scripts/dev/gemv_sweep.py 1,8,16,32,64,128 gemv,umma 4096x4096,11008x4096,8192x8192,28672x8192 > gpurun_out/sweep2.log 2>&1; grep -v relerr gpurun_out/sweep2.log | cut -c1-150
