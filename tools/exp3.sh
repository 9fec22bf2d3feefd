mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mttkrp_gpu.py -q -x -k "tma or engines or baseline" > gpurun_out/tma3.log 2>&1
echo "rc=$?" >> gpurun_out/tma3.log
timeout 600 python tools/sweep.py --shape 1024 1024 1024 --ranks 2000 --rank-tiles 128 256 --block-ks 0 --engines tma --reps 2 --out gpurun_out/sweep_c4.csv > gpurun_out/sweep_c4.log 2>&1
timeout 600 python tools/sweep.py --shape 4096 2048 2048 --ranks 512 --rank-tiles 128 256 --block-ks 0 --engines tma --reps 2 --out gpurun_out/sweep_c5.csv > gpurun_out/sweep_c5.log 2>&1
timeout 600 python tools/sweep.py --shape 512 512 512 --ranks 64 --rank-tiles 0 64 --block-ks 0 --engines auto tma cpasync --reps 3 --out gpurun_out/sweep_c2b.csv > gpurun_out/sweep_c2b.log 2>&1
timeout 600 python tools/sweep.py --shape 128 128 128 128 --ranks 256 --rank-tiles 0 128 256 --block-ks 0 --engines auto tma cpasync --reps 3 --out gpurun_out/sweep_c3.csv > gpurun_out/sweep_c3.log 2>&1
