#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SHIFTADD_CLUSTER_BTAIL=1 timeout 400 python -m pytest tests -m gpu -x -q -k "gemv or config or determin or basis" 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 11008:4096:3 768:768:3"
for rep in 1 2; do
echo "== async tail"; timeout 300 python tools/time_gemv.py --pdl $SH
echo "== barrier tail"; SHIFTADD_CLUSTER_BTAIL=1 timeout 300 python tools/time_gemv.py --pdl $SH
done
bash tools/sweep_mix.sh
SHIFTADD_CLUSTER_BTAIL=1 timeout 300 python tools/time_mix.py 4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3
timeout 900 python tools/bench_extra.py 2>&1 | grep -v Warn | tail -20
