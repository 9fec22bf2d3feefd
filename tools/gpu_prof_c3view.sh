#!/bin/bash
# ncu --set full of the c3 dimension-tree view MTTKRP (16384 x 128 x 128, R = 256, mode 0; KR merge + DMMA).
set -u
TAG=${1:-r02v}
O=gpurun_out
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
  -o /tmp/prof_c3view_$TAG -f python tools/profile_one.py --dims 16384 128 128 --rank 256 --mode 0 --reps 2 > $O/ncu_c3view_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_c3view_$TAG.ncu-rep --tag c3view_$TAG --out $O --aux >> $O/ncu_c3view_$TAG.log 2>&1
echo done
