timeout 600 python scripts/decode_bench.py --layers 4 --reps 2 2>&1 | tail -5
timeout 900 python scripts/decode_bench.py 2>&1 | tail -5
