#!/bin/bash
# Debug build of the library with the kernel profiles compiled in (never the product build):
#   bash tools/build_debug.sh && FLEXQ_LIB=paper_2508_04405_b200/_lib/libflexq_debug.so ...
set -e
cd "$(dirname "$0")/.."
OUT=/tmp/flexq_dbg_obj; mkdir -p $OUT
for f in paper_2508_04405_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       --expt-relaxed-constexpr -DFLEXQ_TC16_TIMELINE=1 -DFLEXQ_TC_TIMELINE_MARKS=1 \
       -c $f -o $OUT/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2508_04405_b200/_lib/libflexq_debug.so $OUT/*.o
echo built paper_2508_04405_b200/_lib/libflexq_debug.so
