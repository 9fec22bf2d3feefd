#!/bin/bash
# Dimension-tree CP-ALS on the GPU: its tests, the CP-ALS suites it touches, a bench pass with the c3 / c5 legs.
set -u
TAG=${1:-dt}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_dimtree_gpu.py tests/test_cpals_gpu.py tests/test_sharded_gpu.py -x -q > $O/pytest_dimtree_$TAG.log 2>&1; echo "rc=$?" >> $O/pytest_dimtree_$TAG.log
timeout 900 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --dfma-steps 1 --gemm-steps 1 --rank-sweep 0 --f32-steps 1 --no-cpu > $O/bench_dimtree_$TAG.json 2> $O/bench_dimtree_$TAG.err; echo "rc=$?" >> $O/bench_dimtree_$TAG.err
echo done
