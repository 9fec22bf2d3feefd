#!/bin/bash
# split-K merge variants at c4: time (ab_lib, c4 only) and DRAM bytes (ncu) of mode 0.
set -u
O=gpurun_out; mkdir -p $O
L=$O/chain_exp2.log
run() {  # env..., splits
  echo "== $1 splits $2" >> $L
  env $1 timeout 300 python tools/profile_one.py --mode 0 --reps 4 --splits $2 2>&1 | grep "mode 0:" | tail -3 >> $L
  env $1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:mttkrp_f64 -s 1 -c 1 python tools/profile_one.py --mode 0 --reps 2 --splits $2 2>&1 | grep -E "dram__|gpu__time" >> $L
}
run "CPK_SPLIT_CHAIN=0" 0
run "CPK_SPLIT_CHAIN=0 CPK_DBG_EPI=4" 0
run "CPK_SPLIT_CHAIN=1" 0
run "CPK_SPLIT_CHAIN=1 CPK_DBG_EPI=1" 0
run "CPK_SPLIT_CHAIN=1 CPK_DBG_EPI=2" 0
run "CPK_SPLIT_CHAIN=1 CPK_DBG_EPI=3" 0
run "CPK_SPLIT_CHAIN=1 CPK_DBG_EPI=2" 256
run "CPK_SPLIT_CHAIN=1 CPK_DBG_EPI=3" 256
run "CPK_SPLIT_CHAIN=0 CPK_DBG_EPI=4" 256
echo done
