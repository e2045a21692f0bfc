timeout 300 python -m pytest tests -x -q -m gpu -k "linear" > gpurun_out/pytest_linear.log 2>&1; tail -2 gpurun_out/pytest_linear.log
timeout 60 python scripts/dev/gemv_trace.py 28672 8192 1 2
timeout 300 python scripts/dev/gemv_sweep.py 1,8,16 > gpurun_out/sweep.log 2>&1; grep -v relerr gpurun_out/sweep.log | grep '"pdl": true'; grep relerr gpurun_out/sweep.log | sort -t: -k5 | tail -1
