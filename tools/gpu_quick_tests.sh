#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_mttkrp_gpu.py tests/test_cpals_gpu.py -q -x -m gpu -k "beyond_five or orders or capi or dten or fuzz" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
echo done
