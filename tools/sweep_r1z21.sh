#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
B="4096:4096:2 11008:4096:3 4096:4096:3 768:768:3"
for m in 3 4; do
echo "== M=$m cluster ring"; timeout 300 python tools/time_gemv.py --pdl --m $m $B 2>&1 | grep -v Warn
echo "== M=$m small-batch split-K"; SHIFTADD_M4_RING=0 timeout 300 python tools/time_gemv.py --pdl --m $m $B 2>&1 | grep -v Warn
done
timeout 300 python tools/bench_extra.py --only llama7b_batch 2>&1 | grep -v Warn | head -5
