#!/bin/bash
# fp16-pair LUT (4 slices per 64 KB): clusters of S/4 (132 SMs at K = 4096) vs the fp32 ring.
cd "$(dirname "$0")/.."
SHIFTADD_LUT16=1 timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== fp32 ring"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== fp16 ring"; SHIFTADD_LUT16=1 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3 2048:2048:3"
echo "== fp32 per-layer"; timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
echo "== fp16 per-layer"; SHIFTADD_LUT16=1 timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
SHIFTADD_LUT16=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 3 --pdl 2>&1 | grep -v Warn | head -12
SHIFTADD_LUT16=1 SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 4096 4096 2 --pdl 2>&1 | grep -v Warn | head -12
