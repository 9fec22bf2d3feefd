#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
for v in 0 1; do
  CPK_KR_MERGE_LAST=$v timeout 600 python tools/kr_last_ab.py > $O/kr_last_ab_$v.json 2> $O/kr_last_ab_$v.err
done
CPK_KR_MERGE_LAST=1 timeout 900 python -m pytest tests/test_mttkrp_gpu.py tests/test_dimtree_gpu.py tests/test_cpals_gpu.py -x -q > $O/kr_last_pytest.log 2>&1; echo "rc=$?" >> $O/kr_last_pytest.log
echo done
