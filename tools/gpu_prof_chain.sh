#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
CPK_SPLIT_CHAIN=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
  -o /tmp/prof_chain -f python tools/profile_one.py --mode 0 --reps 2 --splits 256 > $O/prof_chain.log 2>&1
python tools/ncu_hot.py /tmp/prof_chain.ncu-rep regex:mttkrp 40 > $O/chain_hot.txt 2>&1
python tools/ncu_summary.py /tmp/prof_chain.ncu-rep --tag chain --aux --out $O >> $O/prof_chain.log 2>&1
echo done
