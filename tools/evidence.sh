#!/bin/bash
# The round's GPU evidence in one gpurun call (run from the repo root on the GPU box):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/evidence.sh r2b'
# then, here: python tools/summarize_ncu.py r2b gpurun_out/r2b/launches.csv gpurun_out/r2b/prof_*.ncu-rep
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
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-layers --no-program > $OUT/ncu_launches.log 2>&1
# full captures of the step's kernels: q/k/v fused (kernel 10), o_proj + gate/up concat (3),
# down_proj (8); the LLaMA-2-70B gate/up shape on kernel 8; one persistent program launch (9)
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-layers --no-program"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_cluster_fused -c 2 -o $OUT/prof_fused $B > $OUT/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_cluster_ring -c 2 -o $OUT/prof_cluster $B > $OUT/ncu_cluster.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lut_stream -c 2 -o $OUT/prof_stream $B > $OUT/ncu_stream.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_stream -c 1 -o $OUT/prof_stream70b \
  python tools/prof_gemv.py 28672 8192 3 1 2 > $OUT/ncu_70b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lut_program -c 1 -o $OUT/prof_program \
  python tools/time_program.py --steps 2 > $OUT/ncu_program.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi_end.csv 2>&1
ls -la $OUT
