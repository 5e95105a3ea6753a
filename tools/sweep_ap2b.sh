#!/bin/bash
cd "$(dirname "$0")/.."
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 2048:8192:3 768:768:3"
echo "== K=1"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== K=2"; timeout 300 python tools/time_gemv.py --pdl --apot2 $SH
