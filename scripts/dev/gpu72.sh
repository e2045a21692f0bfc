#!/bin/bash
mkdir -p gpurun_out
for v in old new old new; do
  if [ $v = old ]; then export TRITRUN_LIB=$PWD/scripts/dev/var/k5old/libtritrun.so; else unset TRITRUN_LIB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --sweep "16,32,64,128" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', [(s['batch'], s['ms'], s['speedup_vs_fp16']) for s in d['sweep']])" >> gpurun_out/ab72.txt
done
cat gpurun_out/ab72.txt
unset TRITRUN_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "umma or tq1 or decoder" 2>&1 | tail -3
