#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 300 python tools/bench_extra.py --only llama7b_batch 2>&1 | grep -v Warn | head -5
for m in 5 8 16; do
echo "== M=$m chunks"; timeout 300 python tools/time_gemv.py --pdl --m $m 4096:4096:2 11008:4096:3 2>&1 | grep -v Warn
echo "== M=$m split-K"; SHIFTADD_M4_RING=0 timeout 300 python tools/time_gemv.py --pdl --m $m 4096:4096:2 11008:4096:3 2>&1 | grep -v Warn
done
