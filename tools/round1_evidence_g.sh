#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r1g.json 2>gpurun_out/bench_r1g.err; tail -1 gpurun_out/bench_r1g.json
timeout 900 python tools/bench_extra.py --out gpurun_out/r1g_extra.jsonl 2>&1 | grep -v Warn | tail -20
