#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "umma" 2>&1 | tail -1
for v in base new base new; do
  if [ $v = new ]; then unset TRITRUN_LIB; else export TRITRUN_LIB=$PWD/scripts/dev/var/$v/libtritrun.so; fi
  for shp in "11008 4096 128" "4096 4096 128" "4096 11008 128"; do
    echo "$v $shp $(timeout 120 python scripts/dev/umma_probe.py $shp 0,3 0 2>&1 | grep -o '"us": [0-9.]*' | tr '\n' ' ')"
  done
  echo "$v $(timeout 300 python bench.py --steps 10 --warmup 3 --sweep "64,128" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(s['batch'], s['ms'], s['speedup_vs_fp16']) for s in d['sweep']])")"
done
