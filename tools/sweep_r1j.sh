SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3"
for pb in 8 1 0; do echo "== PREBUILD=$pb"; SHIFTADD_PREBUILD=$pb timeout 120 python tools/time_gemv.py $SH 2>&1 | grep -v Warn; done
for pw in 8 1 0; do echo "== PREWAIT=$pw --pdl"; SHIFTADD_PREWAIT=$pw timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn; done
for pb in 1 0; do
echo "== trace prebuild $pb"; SHIFTADD_PREBUILD=$pb SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py 4096 4096 2 2>&1 | grep -v Warn | head -9
done
