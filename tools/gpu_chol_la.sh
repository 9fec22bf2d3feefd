#!/bin/bash
# Look-ahead chol_small_kernel: solve tests, A/B solve timing vs the previous build, c3 CP-ALS sweep.
set -u
TAG=${1:-r02k}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_solve_gpu.py tests/test_cpals_gpu.py tests/test_dimtree_gpu.py -q -m gpu --timeout 600 > $O/pytest_chol_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_chol_$TAG.log
for lib in paper_2510_14891_b200/_lib/ab/libcpk_b200_prechol.so paper_2510_14891_b200/_lib/libcpk_b200.so; do
  echo "lib $lib" >> $O/solve_ab_$TAG.log
  timeout 300 python tools/solve_bench.py --lib $lib --ranks 32 64 128 192 256 384 --rows 128 1024 --paths kernel --reps 50 >> $O/solve_ab_$TAG.log 2>&1
done
timeout 600 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dfma-steps 0 --gemm-steps 0 --f32-steps 0 --rank-sweep 0 --tree-steps 0 --c5-iters 0 --no-cpu --cpals-iters 10 > $O/bench_c3_$TAG.log 2>&1; echo "rc=$?" >> $O/bench_c3_$TAG.log
echo done
