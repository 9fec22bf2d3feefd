# DMMA vs DFMA consumer sweep over the BASELINE shapes (run under gpurun)
mkdir -p gpurun_out
T=${1:-dmma}
timeout 600 python tools/sweep.py --shape 512 512 512 --ranks 64 --rank-tiles 64 128 --block-ks 0 --engines tma dmma --reps 3 --out gpurun_out/sweep_c2_$T.csv > gpurun_out/sweep_c2_$T.log 2>&1
timeout 600 python tools/sweep.py --shape 128 128 128 128 --ranks 256 --rank-tiles 64 128 256 --block-ks 0 --engines tma dmma --reps 3 --out gpurun_out/sweep_c3_$T.csv > gpurun_out/sweep_c3_$T.log 2>&1
timeout 900 python tools/sweep.py --shape 1024 1024 1024 --ranks 2000 --rank-tiles 64 128 256 --block-ks 0 --engines dmma --reps 2 --out gpurun_out/sweep_c4_$T.csv > gpurun_out/sweep_c4_$T.log 2>&1
timeout 900 python tools/sweep.py --shape 4096 2048 2048 --ranks 512 --rank-tiles 64 128 256 --block-ks 0 --engines dmma --reps 2 --out gpurun_out/sweep_c5_$T.csv > gpurun_out/sweep_c5_$T.log 2>&1
for f in gpurun_out/sweep_c*_$T.agg.csv; do echo "== $f"; cat $f; done
