#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture.
# Usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $OUT/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --dfma-steps 0 --gemm-steps 0 --f32-steps 0 --rank-sweep 0 --cpals-iters 0 --c5-iters 0 --no-cpu > $OUT/ncu_launch_bench_$TAG.log 2>&1
for m in 0 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
    -o $OUT/prof_c4_mode${m}_$TAG -f python tools/profile_one.py --mode $m --reps 2 > $OUT/ncu_full_mode${m}_$TAG.log 2>&1
done
echo done
