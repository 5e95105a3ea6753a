#!/bin/bash
cd "$(dirname "$0")/.."
./tools/probe_clusters.bin
B="4096:11008:2 4096:11008:3 2048:8192:3 8192:8192:2 4096:8192:3"
echo "== default"; timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
echo "== BIGC=1 (stream instead of 4-slot clusters)"; SHIFTADD_CLUSTER_BIGC=1 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
echo "== no cluster"; SHIFTADD_CLUSTER=0 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
