#!/bin/bash
set -u
TAG=${1:-lr}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -q -x -m gpu --timeout 300 > $O/pytest_$TAG.log 2>&1; echo "rc=$?" >> $O/pytest_$TAG.log
timeout 600 python tools/lowrank_sweep.py --ranks 8 16 24 32 40 48 56 64 96 128 > $O/lowrank_new_$TAG.log 2>&1
for i in 1 2; do
timeout 600 python tools/ab_lib.py > $O/ab_new${i}_$TAG.log 2>&1
timeout 600 python tools/ab_lib.py --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_r02base.so > $O/ab_base${i}_$TAG.log 2>&1
done
for rt in 16 32; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
    -o /tmp/prof_c2r16_t${rt}_$TAG -f python tools/profile_one.py --mode 1 --reps 2 --dims 512 512 512 --rank 16 --rank-tile $rt --engine dmma > $O/ncu_c2r16_t${rt}_$TAG.log 2>&1
  python tools/ncu_summary.py /tmp/prof_c2r16_t${rt}_$TAG.ncu-rep --tag $TAG --aux --out $O >> $O/ncu_c2r16_t${rt}_$TAG.log 2>&1
done
echo done
