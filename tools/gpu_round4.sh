#!/bin/bash
# Final round-2 GPU session: tests, smoke, bench, reference arm, launch list, c4 ncu --set full (summarized), NCCL same-GPU probe.
set -u
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
bash tools/gpu_round3.sh $TAG
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_$TAG.log 2>&1; echo "ref rc=$?" >> $O/bench_ref_$TAG.log
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 tools/nccl_same_gpu_probe.py > $O/nccl_probe_$TAG.log 2>&1; echo "rc=$?" >> $O/nccl_probe_$TAG.log
echo done
