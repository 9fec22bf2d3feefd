#!/bin/bash
# split-K chain vs partial copies at c4: time (ab_lib) and DRAM bytes (ncu) per mode.
set -u
O=gpurun_out; mkdir -p $O
L=$O/chain_exp.log
for env in "CPK_SPLIT_CHAIN=0" "CPK_SPLIT_CHAIN=auto"; do
  echo "== $env ab" >> $L
  env $env timeout 300 python tools/ab_lib.py --reps 3 >> $L 2>&1
done
for env in "CPK_SPLIT_CHAIN=0" "CPK_SPLIT_CHAIN=auto"; do
 for sp in 0 256; do
  for m in 0 1; do
   echo "== $env splits $sp mode $m" >> $L
   env $env timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:"mttkrp_f64|splitk" -s 2 -c 2 python tools/profile_one.py --mode $m --reps 2 --splits $sp 2>&1 | grep -E "dram__|gpu__time|lts__t|mttkrp_f64_ws|splitk_reduce|mode" >> $L
  done
 done
done
timeout 600 python -m pytest tests/test_mttkrp_gpu.py tests/test_cpals_gpu.py tests/test_solve_gpu.py -q -x -m gpu > $O/pytest_chain.log 2>&1; echo "rc=$?" >> $O/pytest_chain.log
timeout 600 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --dfma-steps 0 --gemm-steps 0 --f32-steps 0 --rank-sweep 0 --cpals-iters 0 --c5-iters 2 --no-cpu > $O/bench_c5_chain.log 2>&1; echo "rc=$?" >> $O/bench_c5_chain.log
echo done
