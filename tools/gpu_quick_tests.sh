#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_mttkrp_gpu.py -q -x -m gpu -k "tall or landed or streaming or narrow or fuzz or c4_row" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
timeout 300 python tools/ab_lib.py --reps 3 > $O/ab_quick.log 2>&1
echo done
