#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
L=$O/solve_ab.log
for s in default kernel sweep cusolver; do
  if [ $s = default ]; then timeout 300 python tools/cpals_solve_ab.py >> $L 2>&1; else CPK_SOLVE=$s timeout 300 python tools/cpals_solve_ab.py >> $L 2>&1; fi
done
for s in kernel sweep; do CPK_SOLVE=$s timeout 300 python tools/cpals_solve_ab.py --rank 128 >> $L 2>&1; done
for s in kernel sweep; do CPK_SOLVE=$s timeout 300 python tools/cpals_solve_ab.py --rank 64 >> $L 2>&1; done
timeout 300 python tools/solve_bench.py > $O/solve_bench.log 2>&1
echo done
