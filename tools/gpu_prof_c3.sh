mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 2 -c 1 -o gpurun_out/prof_c3_mode1 -f \
  python tools/profile_one.py --mode 1 --reps 3 --dims 128 128 128 128 --rank 256 > gpurun_out/prof_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mttkrp_f64 -s 2 -c 1 -o gpurun_out/prof_c2_mode1 -f \
  python tools/profile_one.py --mode 1 --reps 3 --dims 512 512 512 --rank 64 > gpurun_out/prof_c2.log 2>&1
tail -3 gpurun_out/prof_c3.log
