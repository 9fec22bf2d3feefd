#!/bin/bash
# 4-column micro-blocked diagonal factorization in chol_small_kernel: bits vs the previous build, tests, A/B, c3.
set -u
TAG=${1:-r02q}
O=gpurun_out
mkdir -p $O
for lib in paper_2510_14891_b200/_lib/ab/libcpk_b200_la.so paper_2510_14891_b200/_lib/libcpk_b200.so; do
  timeout 300 python tools/solve_bits.py --lib $lib > $O/solve_bits_$(basename $lib .so)_$TAG.log 2>&1
done
timeout 900 python -m pytest tests/test_solve_gpu.py tests/test_cpals_gpu.py tests/test_dimtree_gpu.py tests/test_sharded_gpu.py -q -m gpu --timeout 600 > $O/pytest_chol_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_chol_$TAG.log
for lib in paper_2510_14891_b200/_lib/ab/libcpk_b200_prechol.so paper_2510_14891_b200/_lib/ab/libcpk_b200_la.so paper_2510_14891_b200/_lib/libcpk_b200.so; do
  echo "lib $lib" >> $O/solve_ab_$TAG.log
  timeout 300 python tools/solve_bench.py --lib $lib --ranks 32 64 128 192 256 384 --rows 128 --paths kernel --reps 100 >> $O/solve_ab_$TAG.log 2>&1
done
timeout 600 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dfma-steps 0 --gemm-steps 0 --f32-steps 0 --rank-sweep 0 --tree-steps 0 --c5-iters 0 --no-cpu --cpals-iters 10 > $O/bench_c3_$TAG.log 2>&1; echo "rc=$?" >> $O/bench_c3_$TAG.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:chol_small -s 3 -c 1 -o /tmp/prof_chol_$TAG -f python tools/solve_bench.py --ranks 256 --rows 128 --paths kernel --reps 2 > $O/ncu_chol_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_chol_$TAG.ncu-rep --tag chol_$TAG --out $O --aux >> $O/ncu_chol_$TAG.log 2>&1
echo done
