#!/bin/bash
# A/B: in-loop push vs push-at-end, prefill depth before griddepcontrol.wait.
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis" 2>&1 | tail -2
SHIFTADD_PUSH_END=1 timeout 300 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis" 2>&1 | tail -2
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
for pe in 0 1; do for kb in 96 200; do
  echo "== PUSH_END=$pe PRE_KB=$kb"; SHIFTADD_PUSH_END=$pe SHIFTADD_PRE_KB=$kb timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done; done; done
for pe in 0 1; do
  echo "== trace PUSH_END=$pe"
  SHIFTADD_PUSH_END=$pe SHIFTADD_PRE_KB=200 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 3 --pdl 2>&1 | grep -v Warn | head -10
done
