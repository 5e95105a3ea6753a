#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -k "ring or small_batch or kernel_choice" 2>&1 | tail -2
for s in "4096 4096 2" "4096 4096 3" "16384 4096 3"; do
  SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -12
done
