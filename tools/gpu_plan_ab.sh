#!/bin/bash
# A/B of the split-count cost model: auto plans and times, previous build vs this one.
set -u
TAG=${1:-r02n}
O=gpurun_out
mkdir -p $O
for rep in 1 2; do
for lib in paper_2510_14891_b200/_lib/ab/libcpk_b200_prechol.so paper_2510_14891_b200/_lib/libcpk_b200.so; do
  timeout 600 python tools/plan_ab.py --lib $lib --reps 10 >> $O/plan_ab_$TAG.log 2>&1
done
done
echo done
