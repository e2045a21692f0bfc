timeout 600 python -m pytest tests -x -q -m gpu -k "tq1" > gpurun_out/pytest_tq1.log 2>&1; tail -15 gpurun_out/pytest_tq1.log
