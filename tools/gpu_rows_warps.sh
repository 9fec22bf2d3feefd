#!/bin/bash
# chol_rows_kernel with 4 / 8 / 16 warps per CTA: bits and factor + apply time.
set -u
TAG=${1:-r02s}
O=gpurun_out
mkdir -p $O
for lib in paper_2510_14891_b200/_lib/libcpk_b200.so paper_2510_14891_b200/_lib/ab/libcpk_b200_rw8.so paper_2510_14891_b200/_lib/ab/libcpk_b200_rw16.so; do
  timeout 300 python tools/solve_bits.py --lib $lib > $O/solve_bits_$(basename $lib .so)_$TAG.log 2>&1
  echo "lib $lib" >> $O/rows_ab_$TAG.log
  timeout 300 python tools/solve_bench.py --lib $lib --ranks 64 128 256 --rows 128 1024 4096 --paths kernel --reps 100 >> $O/rows_ab_$TAG.log 2>&1
done
echo done
