#!/bin/bash
# In-loop DSMEM push reduction + split prefill (x requested before most of the ring): GPU
# tests, prefill-depth sweep on the bench layer mix, traces.
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for kb in 0 24 48 72 96 200; do
  echo "== PRE_KB=$kb"; SHIFTADD_PRE_KB=$kb timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -2
done
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3"
timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
for s in "4096 4096 2" "16384 4096 3"; do
  SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn | head -10
done
timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1
