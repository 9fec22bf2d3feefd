#!/bin/bash
# Low-rank / shared-memory layout experiment: parity, sweep new vs older libs, A/B c2-c4, ncu.
set -u
TAG=${1:-lr}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests/test_mttkrp_gpu.py tests/test_cpals_gpu.py -q -x -m gpu > $O/pytest_$TAG.log 2>&1; echo "rc=$?" >> $O/pytest_$TAG.log
timeout 600 python tools/lowrank_sweep.py > $O/lowrank_new_$TAG.log 2>&1
for L in narrow1 r02base; do
  timeout 600 python tools/lowrank_sweep.py --tiles 16 32 64 --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_$L.so > $O/lowrank_${L}_$TAG.log 2>&1
done
timeout 600 python tools/ab_lib.py > $O/ab_new_$TAG.log 2>&1
timeout 600 python tools/ab_lib.py --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_r02base.so > $O/ab_base_$TAG.log 2>&1
for m in 0 1; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
    -o $O/prof_c2r16_mode${m}_$TAG -f python tools/profile_one.py --mode $m --reps 2 --dims 512 512 512 --rank 16 > $O/ncu_c2r16_mode${m}_$TAG.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
    -o /tmp/prof_c4_mode${m}_$TAG -f python tools/profile_one.py --mode $m --reps 2 > $O/ncu_c4_mode${m}_$TAG.log 2>&1
  python tools/ncu_summary.py /tmp/prof_c4_mode${m}_$TAG.ncu-rep --tag $TAG --aux --out $O >> $O/ncu_c4_mode${m}_$TAG.log 2>&1
  python tools/ncu_lds.py /tmp/prof_c4_mode${m}_$TAG.ncu-rep regex:mttkrp 12 > $O/lds_c4_mode${m}_$TAG.txt 2>&1
done
echo done
