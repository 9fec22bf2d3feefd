#!/bin/bash
# Validation after the chol look-ahead and the split-count model: GPU suite, smoke, full bench, reference arm.
set -u
TAG=${1:-r02o}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $O/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_$TAG.csv \
  python tools/c3_sweep_launches.py > $O/ncu_c3_$TAG.log 2>&1
echo done
