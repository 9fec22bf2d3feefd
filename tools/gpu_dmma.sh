mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mttkrp_gpu.py -q -x -k "dmma or engines_agree" > gpurun_out/dmma_tests.log 2>&1; tail -3 gpurun_out/dmma_tests.log
for cfg in "auto 0" "dmma 128" "dmma 256" "dmma 64"; do set -- $cfg
  echo "== engine $1 rank_tile $2"; timeout 300 python tools/profile_one.py --mode -1 --reps 3 --engine $1 --rank-tile $2 2>&1 | grep -v "^[0-9] {"
done > gpurun_out/dmma_c4.log 2>&1
cat gpurun_out/dmma_c4.log
