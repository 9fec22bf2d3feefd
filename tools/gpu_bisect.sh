#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
run() { echo "== $*" >> $O/bisect3.log; timeout 20 python tools/profile_one.py --reps 2 --dims 512 512 512 --engine dmma "$@" >> $O/bisect3.log 2>&1; echo "rc=$?" >> $O/bisect3.log; }
run --mode 1 --rank 24 --rank-tile 16 --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_dbgFULLNA.so
run --mode 1 --rank 32 --rank-tile 16 --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_dbgFULLNA.so
run --mode 1 --rank 24 --rank-tile 16 --lib paper_2510_14891_b200/_lib/ab/libcpk_b200_swz1.so
timeout 60 compute-sanitizer --tool synccheck python tools/profile_one.py --reps 1 --dims 64 64 64 --rank 24 --rank-tile 16 --engine dmma --mode 1 --splits 1 >> $O/bisect3.log 2>&1
timeout 60 python tools/profile_one.py --reps 1 --dims 64 64 64 --rank 24 --rank-tile 16 --engine dmma --mode 1 --splits 1 >> $O/bisect3.log 2>&1; echo "rc=$?" >> $O/bisect3.log
timeout 60 python tools/profile_one.py --reps 1 --dims 512 64 64 --rank 24 --rank-tile 16 --engine dmma --mode 1 --splits 1 >> $O/bisect3.log 2>&1; echo "rc=$?" >> $O/bisect3.log
timeout 60 python tools/profile_one.py --reps 1 --dims 64 512 64 --rank 24 --rank-tile 16 --engine dmma --mode 1 --splits 1 >> $O/bisect3.log 2>&1; echo "rc=$?" >> $O/bisect3.log
echo done
