#!/bin/bash
# TMA-ring split-K kernel (kernel 4) for large layers: parity, then timing vs the register ring.
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
B="28672:8192:3 8192:28672:3 4096:11008:3 11008:4096:2 8192:8192:2 16384:4096:3"
echo "== register ring"; SHIFTADD_STREAM=0 SHIFTADD_CLUSTER=0 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
for pre in 1 2 4 8; do
  echo "== TMA ring PRE=$pre"; SHIFTADD_STREAM_PRE=$pre SHIFTADD_CLUSTER=0 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
done
echo "== TMA ring no PDL"; SHIFTADD_CLUSTER=0 timeout 300 python tools/time_gemv.py $B 2>&1 | grep -v Warn
