#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_r1i.json 2>gpurun_out/bench_r1i.err; tail -1 gpurun_out/bench_r1i.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r1i.json 2>&1; tail -1 gpurun_out/bench_ref_r1i.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemv_ --csv --log-file gpurun_out/launches_r1i.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_i.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_ -s 0 -c 4 -o gpurun_out/prof_bench_layers_r1i python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_i.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m4_kernel -s 1 -c 1 -o gpurun_out/prof_m4_r1i python tools/prof_gemv.py 11008 4096 3 4 3 > gpurun_out/ncu_m4_i.log 2>&1
timeout 900 python tools/bench_extra.py --out gpurun_out/r1i_extra.jsonl 2>&1 | grep -v Warn | tail -20
ls -la gpurun_out | tail -12
