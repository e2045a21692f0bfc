python scripts/dev/gemv_probe.py 28672 8192 1 0,4096,74,4170
python scripts/dev/gemv_probe.py 4096 4096 1 0,4096
