#!/bin/bash
# Round-2 GPU session: tests, smoke, bench, launch list, c4 ncu --set full (summarized on the box).
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/nvidia-smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.log 2>&1; echo "bench rc=$?" >> $O/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --dfma-steps 0 --gemm-steps 0 --f32-steps 0 --rank-sweep 0 --cpals-iters 0 --c5-iters 0 --no-cpu > $O/ncu_launch_bench_$TAG.log 2>&1
for m in 0 1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 1 -c 1 \
    -o /tmp/prof_c4_mode${m}_$TAG -f python tools/profile_one.py --mode $m --reps 2 > $O/ncu_full_mode${m}_$TAG.log 2>&1
  python tools/ncu_summary.py /tmp/prof_c4_mode${m}_$TAG.ncu-rep --tag $TAG --out $O >> $O/ncu_full_mode${m}_$TAG.log 2>&1
  python tools/ncu_lds.py /tmp/prof_c4_mode${m}_$TAG.ncu-rep regex:mttkrp 8 > $O/lds_c4_mode${m}_$TAG.txt 2>&1
done
du -sh $O
echo done
