#!/bin/bash
# Paper-style reproductions with the round-2 kernels: Table III (tensors A/B, R = 32) and Fig. 4 (GFLOP/s vs R).
set -u
mkdir -p gpurun_out
bash tools/gpu_table3.sh > gpurun_out/table3_run.log 2>&1
timeout 900 python tools/fig4.py --out gpurun_out/r02_fig4_c2.csv > gpurun_out/fig4.log 2>&1
echo done
