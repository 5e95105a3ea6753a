#!/bin/bash
# Cluster kernel TMA prefetch stage (first P items per warp), stream kernel trace.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== base"; (cd _base && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== PREF=1"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== PREF=0"; SHIFTADD_PREF=0 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3"
timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
for s in "4096 4096 2" "16384 4096 3"; do
  SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -10
done
SHIFTADD_STREAM_TRACE=1 timeout 120 python tools/trace_stream.py 28672 8192 3 --pdl 2>&1 | grep -v Warn
SHIFTADD_STREAM_TRACE=1 SHIFTADD_STREAM_LOADS_ONLY=1 timeout 120 python tools/trace_stream.py 28672 8192 3 --pdl 2>&1 | grep -v Warn
