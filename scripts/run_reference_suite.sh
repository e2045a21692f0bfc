#!/bin/bash
# Run the reference's OWN test suite with this repo's CUDA kernels as its default backend.
# Needs the reference installed in baseline/_ref (pip install --target baseline/_ref)
# and its tests next to it (copied from /root/reference/pkg/tests when that exists).
set -u
cd "$(dirname "$0")/.."
if [ -d /root/reference/pkg/tests ] && [ ! -d baseline/_ref/tritpack_tests ]; then
  cp -r /root/reference/pkg/tests baseline/_ref/tritpack_tests
fi
PYTHONPATH="$PWD/tests:$PWD:$PWD/baseline/_ref" TRITPACK_BACKEND=cuda python -m pytest -q -p ref_cuda_plugin -p no:cacheprovider \
  --rootdir baseline/_ref baseline/_ref/tritpack_tests "$@"
