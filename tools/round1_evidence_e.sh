#!/bin/bash
# Round-1 evidence, cluster kernel: GPU tests, bench line, ncu launch list + full capture of
# the four bench layers, extra configs.  Outputs under gpurun_out/ (summarised into profiles/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1e.json 2>gpurun_out/bench_r1e.err; tail -1 gpurun_out/bench_r1e.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemv_ --csv --log-file gpurun_out/launches_r1e.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_ -s 0 -c 4 -o gpurun_out/prof_bench_layers_r1e python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c.log 2>&1
timeout 900 python tools/bench_extra.py --out gpurun_out/r1e_extra.jsonl 2>&1 | grep -v Warn | tail -20
ls -la gpurun_out | tail -10
