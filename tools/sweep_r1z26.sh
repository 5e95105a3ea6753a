#!/bin/bash
cd "$(dirname "$0")/.."
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== no prefetch"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
  echo "== translation prefetch"; TM_PREFETCH=1 timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
