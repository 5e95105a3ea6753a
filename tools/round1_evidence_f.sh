#!/bin/bash
# Round-1 evidence, TMA-ring kernels: GPU tests, bench line, ncu launch list + full capture of
# the four bench layers and of the 70B stream kernel, extra configs.  Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1f.json 2>gpurun_out/bench_r1f.err; tail -1 gpurun_out/bench_r1f.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemv_ --csv --log-file gpurun_out/launches_r1f.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_ -s 0 -c 4 -o gpurun_out/prof_bench_layers_r1f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_f.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stream -s 1 -c 1 -o gpurun_out/prof_stream_70b_r1f python tools/prof_gemv.py 28672 8192 3 1 3 > gpurun_out/ncu_stream_f.log 2>&1
SHIFTADD_STREAM_TRACE=1 timeout 120 python tools/trace_stream.py 28672 8192 3 --pdl 2>&1 | grep -v Warn
timeout 900 python tools/bench_extra.py --out gpurun_out/r1f_extra.jsonl 2>&1 | grep -v Warn | tail -20
ls -la gpurun_out | tail -12
