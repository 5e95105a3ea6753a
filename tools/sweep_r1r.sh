#!/bin/bash
# cluster-pair M=1 kernel: parity + timing against the split-K kernel
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 2048:8192:3 11008:4096:3 4096:11008:2 768:768:3"
echo "== pair --pdl"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== splitk --pdl"; timeout 300 python tools/time_gemv.py --pdl --splitk $SH
echo "== pair no pdl"; timeout 300 python tools/time_gemv.py $SH
