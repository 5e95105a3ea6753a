#!/bin/bash
# The round's GPU evidence in one gpurun call (run from the repo root on the GPU box):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/evidence.sh r2a'
# then, here: python tools/summarize_ncu.py r2a gpurun_out/r2a/launches.csv gpurun_out/r2a/prof_*.ncu-rep
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi_start.csv 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2>&1
# launch list of two bench steps (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-layers > $OUT/ncu_launches.log 2>&1
# full captures: the first kernel-8 launches of a step (block 0 q/k/v fused, down; block 1 q/k/v)
# and the first cluster-kernel launches (block 0 o_proj, gate/up concatenated)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lut_stream -c 3 -o $OUT/prof_stream \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-layers > $OUT/ncu_stream.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_cluster_ring -c 2 -o $OUT/prof_cluster \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-layers > $OUT/ncu_cluster.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi_end.csv 2>&1
ls -la $OUT
