#!/bin/bash
# tuning builds: the main objects with one source recompiled under other
# macro settings -> build/variants/<name>/libspechp_b200.so
#   tools/build_variants.sh <source.cu> name:flags [name:flags ...]
set -e
cd "$(dirname "$0")/../paper_1906_03489_b200/csrc"
make -j8 > /dev/null
src=$1; shift
obj=${src%.cu}.o
FL="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  d=../../build/variants/$name
  mkdir -p $d
  nvcc $FL $flags -c $src -o $d/$obj &
done
wait
for v in "$@"; do
  name=${v%%:*}
  d=../../build/variants/$name
  objs=$(ls ../../build/csrc/*.o | grep -v "/$obj")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libspechp_b200.so $objs $d/$obj
done
