timeout 300 python -m pytest tests -x -q -m gpu -k "pre_fused or decoder" > gpurun_out/p.log 2>&1; tail -2 gpurun_out/p.log; grep -E "^E " gpurun_out/p.log | head -5
timeout 300 python scripts/decode_bench.py --reps 3 | tail -1
