#!/bin/bash
set -u
O=gpurun_out; mkdir -p $O
for r in 16 64 256; do timeout 300 python tools/cpals_graph_cost.py --rank $r >> $O/graph_cost.log 2>&1; done
CPK_SOLVE=sweep timeout 300 python tools/cpals_graph_cost.py --rank 256 >> $O/graph_cost.log 2>&1
timeout 300 python tools/cpals_graph_cost.py --rank 64 --dims 256 256 256 >> $O/graph_cost.log 2>&1
echo done
