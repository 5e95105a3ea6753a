#!/bin/bash
# 4 seeded accumulation chains per plane (no 0+v adds) vs the committed 2-chain loop (_base2).
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== before"; (cd _base2 && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== after"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
B="28672:8192:3 8192:28672:3 16384:4096:3"
echo "== before"; (cd _base2 && timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn)
echo "== after"; timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
