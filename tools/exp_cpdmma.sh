mkdir -p gpurun_out
timeout 900 python tools/sweep.py --shape 1024 1024 1024 --ranks 2000 --rank-tiles 64 128 --block-ks 0 --engines dmma cpdmma --reps 2 --out gpurun_out/sweep_c4_cpdmma.csv > gpurun_out/sweep_c4_cpdmma.log 2>&1
timeout 900 python tools/sweep.py --shape 1023 1024 1024 --ranks 2000 --rank-tiles 64 128 --block-ks 0 --engines cpdmma cpasync --reps 2 --out gpurun_out/sweep_odd_cpdmma.csv > gpurun_out/sweep_odd_cpdmma.log 2>&1
timeout 900 python tools/sweep.py --shape 401 201 12 501 --ranks 32 --rank-tiles 32 64 --block-ks 0 --engines cpdmma cpasync --reps 3 --out gpurun_out/sweep_A_cpdmma.csv > gpurun_out/sweep_A_cpdmma.log 2>&1
for f in gpurun_out/sweep_*cpdmma.agg.csv; do echo "== $f"; cat $f; done
