timeout 300 python -m pytest tests -x -q -m gpu -k "umma_ksplit or umma_vs_oracle" > gpurun_out/p.log 2>&1; tail -1 gpurun_out/p.log
timeout 300 python scripts/dev/gemv_sweep.py 16,64,128 umma 4096x4096,11008x4096,8192x8192,28672x8192 2>&1 | grep -v relerr
