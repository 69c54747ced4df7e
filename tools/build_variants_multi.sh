#!/bin/bash
# tuning builds recompiling SEVERAL sources under other macro settings
# (e.g. a geometry layout shared by producers and consumers)
#   SRCS="misc.cu solver.cu hex_helm.cu hex_helm1.cu hex_helm2.cu" tools/build_variants_multi.sh name:flags ...
# The variant libraries land in build/variants/<name>/ (selected at run time
# with SPHP_LIBRARY_VARIANT=<name>); .gpurunignore keeps that directory off
# the GPU box, so drop its build/variants/ line while A/B-ing and restore it.
set -e
cd "$(dirname "$0")/../paper_1906_03489_b200/csrc"
make -j8 > /dev/null
FL="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  d=../../build/variants/$name
  mkdir -p $d
  for src in $SRCS; do
    nvcc $FL $flags -c $src -o $d/${src%.cu}.o &
  done
done
wait
for v in "$@"; do
  name=${v%%:*}
  d=../../build/variants/$name
  objs=""
  for o in ../../build/csrc/*.o; do
    b=$(basename $o)
    if [ -f $d/$b ]; then objs="$objs $d/$b"; else objs="$objs $o"; fi
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libspechp_b200.so $objs
done
