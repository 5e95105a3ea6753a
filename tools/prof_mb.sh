timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tiled_mb -s 2 -c 1 -o gpurun_out/prof_mb4_fc1 python tools/prof_gemv.py 16384 4096 3 4 3 > gpurun_out/ncu_mb.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tiled_mb -s 2 -c 1 -o gpurun_out/prof_mb16_fc1 python tools/prof_gemv.py 16384 4096 3 16 3 >> gpurun_out/ncu_mb.log 2>&1
tail -3 gpurun_out/ncu_mb.log
