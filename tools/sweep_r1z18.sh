#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1h.json 2>gpurun_out/bench_r1h.err; tail -1 gpurun_out/bench_r1h.json; tail -3 gpurun_out/bench_r1h.err
