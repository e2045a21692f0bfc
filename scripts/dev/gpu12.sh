timeout 300 python -m pytest tests -x -q -m gpu -k "umma" > gpurun_out/pytest_umma.log 2>&1; tail -1 gpurun_out/pytest_umma.log
timeout 120 python scripts/dev/umma_probe.py 18944 8192 16 0,1,2,3
timeout 120 python scripts/dev/umma_probe.py 28672 8192 16 0
timeout 120 python scripts/dev/umma_probe.py 28672 8192 128 0
timeout 120 python scripts/dev/umma_probe.py 4096 4096 16 0
