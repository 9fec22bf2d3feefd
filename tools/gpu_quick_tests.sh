#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_bench.py -q -x -m gpu > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
echo done
