#!/bin/bash
cd "$(dirname "$0")/.."
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "small_batch or workspace or wider or bad or apot2 or canonical" 2>&1 | tail -2
for m in 2 3 4 8 16; do timeout 300 python tools/time_gemv.py --pdl --m $m 16384:4096:3 4096:4096:2; done
timeout 600 python tools/bench_extra.py --only llama7b_batch 2>&1 | grep -v Warn | tail -6
