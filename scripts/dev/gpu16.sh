timeout 300 python -m pytest tests -x -q -m gpu -k "decoder" > gpurun_out/pytest_dec.log 2>&1; tail -3 gpurun_out/pytest_dec.log
timeout 900 python scripts/decode_bench.py 2>&1 | tail -2
