#!/bin/bash
# Re-establish state after a container restore: GPU tests, bench line, per-phase traces.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ls -la MEASURED_PEAKS.json 2>&1; cat MEASURED_PEAKS.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1f.json 2>gpurun_out/bench_r1f.err; tail -1 gpurun_out/bench_r1f.json
for s in "4096 4096 2" "4096 4096 3" "16384 4096 2" "16384 4096 3"; do
  SHIFTADD_CLUSTER_TRACE=1 timeout 120 python tools/trace_cluster.py $s --pdl 2>&1 | grep -v Warn
done
