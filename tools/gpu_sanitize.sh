#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $O/sanitize_${tool}_r02.log 2>&1; echo "rc=$?" >> $O/sanitize_${tool}_r02.log
done
echo done
