#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "umma or tq1" 2>&1 | tail -1
for v in base new base new; do
  if [ $v = new ]; then unset TRITRUN_LIB; else export TRITRUN_LIB=$PWD/scripts/dev/var/$v/libtritrun.so; fi
  echo "$v $(timeout 300 python bench.py --steps 10 --warmup 3 --sweep "16,32,64,128" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(s['batch'], s['ms'], s['speedup_vs_fp16']) for s in d['sweep']], d['tq1_8192x8192'])")"
done
