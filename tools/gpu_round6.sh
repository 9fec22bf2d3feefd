#!/bin/bash
# Round-2 final validation after the dimension tree: full GPU suite, smoke, bench, reference arm, launch list,
# c4 ncu --set full (summarized on the box), sanitizers on the small cases.
set -u
TAG=${1:-r02h}
O=gpurun_out
mkdir -p $O
bash tools/gpu_round3.sh $TAG
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> $O/bench_ref_$TAG.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $O/sanitize_${tool}_$TAG.log 2>&1; echo "rc=$?" >> $O/sanitize_${tool}_$TAG.log
done
echo done
