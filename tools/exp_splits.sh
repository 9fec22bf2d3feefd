# DRAM bytes vs split count for the c4 DMMA kernel (mode 0 and 1)
mkdir -p gpurun_out
for m in 0 1; do for s in 15 37 74 148; do
  echo "== mode $m splits $s"
  timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:mttkrp_f64_ws python tools/profile_one.py --mode $m --reps 1 --splits $s 2>&1 | grep -E "dram__|gpu__time|lts__t|mode $m:"
done; done > gpurun_out/exp_splits.log 2>&1
cat gpurun_out/exp_splits.log
