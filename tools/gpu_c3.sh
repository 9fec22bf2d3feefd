mkdir -p gpurun_out
timeout 600 python tools/sweep.py --shape 128 128 128 128 --ranks 256 --rank-tiles 128 --block-ks 0 --engines dmma --splits 0 37 74 148 296 --reps 3 --out gpurun_out/sweep_c3_splits.csv > gpurun_out/sweep_c3_splits.log 2>&1
cat gpurun_out/sweep_c3_splits.agg.csv
