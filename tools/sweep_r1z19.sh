#!/bin/bash
cd "$(dirname "$0")/.."
for m in 1 2 4 8 16; do
  echo "== M=$m"; timeout 300 python tools/time_gemv.py --pdl --m $m 4096:4096:2 11008:4096:3 4096:11008:2 22016:4096:3 2>&1 | grep -v Warn
done
