mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f32 -s 3 -c 1 -o gpurun_out/prof_f32_mode1 -f \
  python tools/f32_bench.py --reps 2 > gpurun_out/prof_f32.log 2>&1
tail -2 gpurun_out/prof_f32.log
