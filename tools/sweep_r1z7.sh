#!/bin/bash
# TMA ring: pure streaming rate (no lookups) vs product; ncu full capture of kernel 4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="28672:8192:3 8192:28672:3"
echo "== loads only"; SHIFTADD_STREAM_LOADS_ONLY=1 SHIFTADD_STREAM_PRE=1 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
echo "== product"; SHIFTADD_STREAM_PRE=1 timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream -s 1 -c 1 -o gpurun_out/prof_stream_70b python tools/prof_gemv.py 28672 8192 3 1 3 > gpurun_out/ncu_stream.log 2>&1
tail -3 gpurun_out/ncu_stream.log
