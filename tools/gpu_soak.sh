#!/bin/bash
# Full GPU suite twice + smoke (flakiness check).
set -u
O=gpurun_out; mkdir -p $O
for i in 1 2; do
  timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $O/soak_$i.log 2>&1; echo "rc=$?" >> $O/soak_$i.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/soak_smoke.log 2>&1; echo "rc=$?" >> $O/soak_smoke.log
echo done
