#!/bin/bash
# Dev A/B: build libtritrun.so with extra -D flags into scripts/dev/ab/<name>/ (load with TRITRUN_LIB=...)
set -e
name=$1; shift
cd "$(dirname "$0")/../../paper_2506_23025_b200"
out=../scripts/dev/ab/$name; mkdir -p $out/obj
for f in csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I../include "$@" -c -o $out/obj/$b.o $f &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libtritrun.so $out/obj/*.o -lcuda
rm -rf $out/obj
echo built $out/libtritrun.so
