#!/bin/bash
# Final session: gpu_round4 (tests, smoke, bench, reference arm, launch list, ncu) + sanitizers.
set -u
TAG=${1:-r02}
bash tools/gpu_round4.sh $TAG
bash tools/gpu_sanitize.sh
echo done
