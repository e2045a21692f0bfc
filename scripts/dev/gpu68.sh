#!/bin/bash
for v in base preall pre8; do
  if [ $v = base ]; then unset TRITRUN_LIB; else export TRITRUN_LIB=$PWD/scripts/dev/var/$v/libtritrun.so; fi
  echo "== $v" >> gpurun_out/ab68.txt
  for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --sweep "" --cpu-seconds 0.1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_us'])" >> gpurun_out/ab68.txt; done
  timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1 >> gpurun_out/ab68.txt
done
