#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
L=$O/graph_r512.log
timeout 300 python tools/cpals_graph_cost.py --rank 512 --dims 512 256 256 >> $L 2>&1
CPK_SWEEP_CTAS=0 timeout 300 python tools/cpals_graph_cost.py --rank 512 --dims 512 256 256 >> $L 2>&1
timeout 300 python tools/cpals_graph_cost.py --rank 300 --dims 128 128 128 128 >> $L 2>&1
CPK_SWEEP_CTAS=0 timeout 300 python tools/cpals_graph_cost.py --rank 300 --dims 128 128 128 128 >> $L 2>&1
echo done
