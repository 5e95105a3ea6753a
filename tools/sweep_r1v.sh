#!/bin/bash
cd "$(dirname "$0")/.."
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 2
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 16384 4096 2 --pdl
SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py 4096 4096 2
