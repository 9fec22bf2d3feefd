#!/bin/bash
# c4 split count A/B with the current kernel (per-mode ms, best of 4).
set -u
O=gpurun_out; mkdir -p $O
L=$O/splits2.log
for sp in 0 111 148 185 222 296; do
  for m in 0 1; do
    echo "== splits $sp mode $m" >> $L
    timeout 300 python tools/profile_one.py --mode $m --reps 5 --splits $sp 2>&1 | grep "mode $m:" | sort -t: -k2 -n | head -2 >> $L
  done
done
echo done
