#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -x -k "gemv or config or determin or basis or fused or misaligned or symmetry" 2>&1 | tail -2
for s in "4096 4096 2" "16384 4096 3"; do SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -11; done
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
