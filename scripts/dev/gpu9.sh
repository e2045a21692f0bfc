timeout 600 python -m pytest tests -x -q -m gpu -k "umma" > gpurun_out/pytest_umma.log 2>&1; tail -15 gpurun_out/pytest_umma.log
