#!/bin/bash
# Stream kernel: fewer owner CTAs (non-owners leave early; the next call's CTAs take their SMs).
cd "$(dirname "$0")/.."
timeout 300 python -m pytest tests -m gpu -x -q -k "parity or tma or determin" 2>&1 | tail -2
SHIFTADD_STREAM_OWNERS=32 timeout 300 python -m pytest tests -m gpu -x -q -k "tma or llama70b or 4736 or 4700 or 2400" 2>&1 | tail -2
B="28672:8192:3 8192:28672:3 4096:11008:2"
for o in 0 16 32 64; do
  echo "== OWNERS=$o"; SHIFTADD_STREAM_OWNERS=$o timeout 300 python tools/time_gemv.py --pdl $B 2>&1 | grep -v Warn
done
M="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
timeout 300 python tools/time_mix.py $M 2>&1 | grep -v Warn | tail -1
