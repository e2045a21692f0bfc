#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "decoder or greedy" > gpurun_out/t77.txt 2>&1; tail -2 gpurun_out/t77.txt
for v in old new old new; do
  if [ $v = new ]; then unset TRITRUN_LIB; else export TRITRUN_LIB=$PWD/scripts/dev/var/attnold/libtritrun.so; fi
  echo "$v $(timeout 300 python scripts/dev/decode_parts.py 2>&1 | tail -1)"
done
