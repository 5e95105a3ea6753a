mkdir -p gpurun_out
timeout 900 python tools/bench_extra.py --out gpurun_out/r1_extra.jsonl 2>&1 | grep -v Warn | tail -20
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemv_tiled --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_tiled -s 0 -c 4 -o gpurun_out/prof_bench_layers_r1b python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_b.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r1b.json 2>gpurun_out/bench_r1b.err; tail -1 gpurun_out/bench_r1b.json
ls -la gpurun_out | tail -8
