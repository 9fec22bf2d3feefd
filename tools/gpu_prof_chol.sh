#!/bin/bash
# ncu --set full of the one-CTA Cholesky (chol_small_kernel) at R = 256; SASS-level stall samples for profiles/r02_chol_small.md
set -u
O=gpurun_out; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_small -s 2 -c 1 -o /tmp/prof_chol -f \
  python tools/solve_bench.py --ranks 256 --rows 128 --paths kernel --reps 3 > $O/prof_chol.log 2>&1
ncu -i /tmp/prof_chol.ncu-rep --page source --csv --print-source cuda -k regex:chol_small > $O/chol_source.csv 2>&1
ncu -i /tmp/prof_chol.ncu-rep --page source --csv --print-source sass -k regex:chol_small > /tmp/chol_sass.csv 2>&1
head -c 3000000 /tmp/chol_sass.csv > $O/chol_sass.csv
echo done
