#!/bin/bash
# x staged by the bulk-copy engine (TMA) vs LSU loads; push-at-end for 4-slot CTAs.
cd "$(dirname "$0")/.."
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 4096:11008:2 768:768:3"
SHIFTADD_X_TMA=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
  echo "== base"; (cd _base && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== new"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== new X_TMA"; SHIFTADD_X_TMA=1 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
echo "== new per-layer"; timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
echo "== new X_TMA per-layer"; SHIFTADD_X_TMA=1 timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
for s in "4096 4096 2" "16384 4096 3"; do
  SHIFTADD_X_TMA=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -10
done
