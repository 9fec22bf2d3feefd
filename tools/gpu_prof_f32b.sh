#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f32 -s 3 -c 1 -o /tmp/prof_f32 -f \
  python tools/f32_bench.py --reps 2 > $O/prof_f32b.log 2>&1
python tools/ncu_summary.py /tmp/prof_f32.ncu-rep --tag f32b --aux --out $O >> $O/prof_f32b.log 2>&1
python tools/ncu_lds.py /tmp/prof_f32.ncu-rep regex:mttkrp_f32 30 > $O/f32_lds.txt 2>&1
python tools/ncu_hot.py /tmp/prof_f32.ncu-rep regex:mttkrp_f32 40 > $O/f32_hot.txt 2>&1
echo done
