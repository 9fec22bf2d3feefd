#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
L=$O/solve_ctas.log
timeout 300 python tools/cpals_solve_ab.py >> $L 2>&1
for c in 1 2 4 8; do echo "ctas $c" >> $L; CPK_SOLVE=sweep CPK_SWEEP_CTAS=$c timeout 300 python tools/cpals_solve_ab.py >> $L 2>&1; done
for c in 1 2; do echo "ctas $c R128" >> $L; CPK_SOLVE=sweep CPK_SWEEP_CTAS=$c timeout 300 python tools/cpals_solve_ab.py --rank 128 >> $L 2>&1; done
echo "kernel R128" >> $L; timeout 300 python tools/cpals_solve_ab.py --rank 128 >> $L 2>&1
echo "c5-like R512 default" >> $L; timeout 300 python tools/cpals_solve_ab.py --rank 512 --dims 512 256 256 >> $L 2>&1
for c in 1 2 4 8 16; do echo "ctas $c R512" >> $L; CPK_SWEEP_CTAS=$c timeout 300 python tools/cpals_solve_ab.py --rank 512 --dims 512 256 256 >> $L 2>&1; done
echo done
