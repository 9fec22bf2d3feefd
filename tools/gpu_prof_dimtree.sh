#!/bin/bash
# ncu evidence for the dimension-tree sweep: launch list (per-kernel time + DRAM bytes) of one c5-proxy
# sweep (1024x2048x2048, R=512: W_G = 17.2 GB, as at c5) and of c3, then --set full of the contraction.
set -u
TAG=${1:-dt}
O=gpurun_out
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/dt_launch_c5p_$TAG.csv \
  python tools/dimtree_sweep.py --dims 1024,2048,2048 --rank 512 --iters 1 > $O/dt_c5p_$TAG.log 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/dt_launch_c3_$TAG.csv \
  python tools/dimtree_sweep.py --dims 128,128,128,128 --rank 256 --iters 1 > $O/dt_c3_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dimtree_contract -c 2 \
  -o /tmp/prof_dt_contract_$TAG python tools/dimtree_sweep.py --dims 1024,2048,2048 --rank 512 --iters 1 \
  > $O/dt_full_$TAG.log 2>&1
python tools/ncu_summary.py /tmp/prof_dt_contract_$TAG.ncu-rep --tag $TAG --aux --out $O >> $O/dt_full_$TAG.log 2>&1
echo done
