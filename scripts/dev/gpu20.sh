timeout 600 python -m pytest tests -x -q -m gpu -k "gemv or linear" > gpurun_out/p.log 2>&1; tail -2 gpurun_out/p.log
timeout 300 python scripts/dev/gemv_sweep.py 1,4 gemv 4096x4096,11008x4096,4096x11008,28672x8192 2>&1 | grep -v relerr
