#!/bin/bash
# bulk-copy size per stage: whole stage (16 items) vs 4 / 1 items per copy.
cd "$(dirname "$0")/.."
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do for sp in 0 4 1; do
  echo "== SPLIT=$sp"; SHIFTADD_RING_SPLIT=$sp timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done; done
SHIFTADD_RING_SPLIT=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 4096 4096 2 --pdl 2>&1 | grep -v Warn | head -11
