#!/bin/bash
# TMA ring: time vs size (fixed overhead vs streaming rate), loads-only and product.
cd "$(dirname "$0")/.."
B="14336:8192:3 28672:8192:3 57344:8192:3 28672:8192:2"
echo "== loads only"; SHIFTADD_STREAM_LOADS_ONLY=1 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
echo "== product"; timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
echo "== register ring"; SHIFTADD_STREAM=0 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
