#!/bin/bash
# exponent tiles copied once per CTA (one bulk copy per slice) instead of one per stage.
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests -m gpu -q -x -k "gemv or config or determin or basis or fused or misaligned or symmetry or colwise" 2>&1 | tail -2
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for rep in 1 2; do
  echo "== prev"; (cd _prev && timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1)
  echo "== exps up front"; timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
done
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3"
echo "== prev"; (cd _prev && timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn)
echo "== exps up front"; timeout 300 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
