#!/bin/bash
# x by TMA with small pre-wait prefill: does x still queue?  Split-K variants on 70B shapes.
cd "$(dirname "$0")/.."
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for kb in 0 24 48 1024; do
  echo "== X_TMA PRE_KB=$kb"
  SHIFTADD_X_TMA=1 SHIFTADD_PRE_KB=$kb timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  SHIFTADD_X_TMA=1 SHIFTADD_PRE_KB=$kb SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 3 --pdl 2>&1 | grep -v Warn | sed -n 2,7p
done
B="28672:8192:3 8192:28672:3 4096:11008:2 11008:4096:3"
echo "== split-K default"; SHIFTADD_CLUSTER=0 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
for v in 0 3; do for ps in 1 2; do
  echo "== split-K VARIANT=$v PER_SM=$ps"; SHIFTADD_CLUSTER=0 SHIFTADD_VARIANT=$v SHIFTADD_PER_SM=$ps timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
done; done
echo "== base 4096x11008"; (cd _base && timeout 300 python tools/time_gemv.py --pdl 4096:11008:2 2>&1 | grep -v Warn)
echo "== new PUSH_END=0 4096x11008"; SHIFTADD_PUSH_END=0 timeout 300 python tools/time_gemv.py --pdl 4096:11008:2 2>&1 | grep -v Warn
