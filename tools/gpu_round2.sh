#!/bin/bash
# Round-2 GPU session: gpu_round.sh plus the reference arm.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.log
bash tools/gpu_round.sh $TAG
