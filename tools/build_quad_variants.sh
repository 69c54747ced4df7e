#!/bin/bash
# quad-kernel tuning builds: the main objects with quad.cu recompiled under
# other budgets / stage counts -> build/variants/<name>/libspechp_b200.so
set -e
cd "$(dirname "$0")/../paper_1906_03489_b200/csrc"
make -j8 > /dev/null
FL="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr"
for v in "b40:-DSPHP_QUAD_BUDGET=40960" "b56:-DSPHP_QUAD_BUDGET=57344" "b100:-DSPHP_QUAD_BUDGET=102400" \
         "n2b56:-DSPHP_QUAD_NST=2 -DSPHP_QUAD_BUDGET=57344" "n2b40:-DSPHP_QUAD_NST=2 -DSPHP_QUAD_BUDGET=40960" \
         "n2b74:-DSPHP_QUAD_NST=2"; do
  name=${v%%:*}; flags=${v#*:}
  d=../../build/variants/$name
  mkdir -p $d
  nvcc $FL $flags -c quad.cu -o $d/quad.o &
done
wait
for d in ../../build/variants/*/; do
  objs=$(ls ../../build/csrc/*.o | grep -v "/quad.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libspechp_b200.so $objs $d/quad.o
done
ls ../../build/variants
