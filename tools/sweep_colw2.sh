#!/bin/bash
cd "$(dirname "$0")/.."
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 4096:2048:3 768:768:3"
echo "== rowwise"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== colwise"; timeout 300 python tools/time_gemv.py --pdl --colwise $SH
