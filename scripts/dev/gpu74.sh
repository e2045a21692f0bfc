#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "umma" > gpurun_out/t74.txt 2>&1; tail -3 gpurun_out/t74.txt
for shp in "11008 4096 128" "4096 4096 128" "4096 11008 128" "11008 4096 64" "11008 4096 32"; do
  timeout 120 python scripts/dev/umma_probe.py $shp 0,4 0 >> gpurun_out/p74.txt 2>&1
done
grep -o '"rows.*' gpurun_out/p74.txt
timeout 300 python bench.py --steps 10 --warmup 3 --sweep "16,32,64,128" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(s['batch'], s['ms'], s['speedup_vs_fp16']) for s in d['sweep']])"
