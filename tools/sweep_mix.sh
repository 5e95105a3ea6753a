#!/bin/bash
cd "$(dirname "$0")/.."
A2=4096:4096:2; A3=4096:4096:3; F2=16384:4096:2; F3=16384:4096:3
for m in "$A2" "$A3" "$F2" "$F3" "$A2 $A2" "$A2 $A3" "$F2 $F3" "$A2 $F2" "$A2 $A3 $F2 $F3" "$A2 $A2 $F2 $F2"; do
  timeout 300 python tools/time_mix.py $m
done
timeout 300 python tools/time_mix.py --nopdl $A2 $A3 $F2 $F3
SHIFTADD_CLUSTER_HALF=0 timeout 300 python tools/time_mix.py $A2 $A3 $F2 $F3
