timeout 400 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_all.log 2>&1; tail -2 gpurun_out/pytest_all.log
timeout 300 python scripts/dev/gemv_sweep.py 1,4,8 auto 3072x9216,4096x11008 2>&1 | grep -v relerr
