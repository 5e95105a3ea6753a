# Round-1 evidence run: tests, bench (default + reference arm), ncu launch list + full captures.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; cat gpurun_out/bench_r1.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1.json 2>&1; cat gpurun_out/bench_ref_r1.json | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tiled -s 4 -c 1 -o gpurun_out/prof_fc1_q3_r1 python tools/prof_gemv.py 16384 4096 3 1 6 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tiled -s 4 -c 1 -o gpurun_out/prof_attn_q2_r1 python tools/prof_gemv.py 4096 4096 2 1 6 >> gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
