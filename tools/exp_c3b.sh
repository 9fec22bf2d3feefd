# c3 per-mode times (auto plan) + ncu of modes 0 and 3 (cold-cache, for stall comparison)
mkdir -p gpurun_out
timeout 300 python tools/profile_one.py --mode -1 --reps 4 --dims 128 128 128 128 --rank 256 > gpurun_out/c3b_times.log 2>&1
for m in 0 3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 2 -c 1 -o gpurun_out/prof_c3_mode$m -f \
  python tools/profile_one.py --mode $m --reps 3 --dims 128 128 128 128 --rank 256 > gpurun_out/prof_c3_m$m.log 2>&1
done
cat gpurun_out/c3b_times.log
