#!/bin/bash
cd "$(dirname "$0")/.."
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
echo "== prev"; (cd _prev && timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn)
echo "== head"; timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
done
