#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests/test_mttkrp_gpu.py tests/test_cpals_gpu.py -q -x -m gpu > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
for i in 1 2; do
timeout 300 python tools/ab_lib.py --reps 3 > $O/ab_new_$i.log 2>&1
timeout 300 python tools/ab_lib.py --reps 3 --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_fold.so > $O/ab_fold_$i.log 2>&1
done
timeout 300 python tools/lowrank_sweep.py --ranks 16 32 64 --tiles 16 32 64 > $O/lowrank_b1.log 2>&1
echo done
