timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2"
echo "== default --pdl"; timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
echo "== M=4 --pdl"; timeout 120 python tools/time_gemv.py --pdl --m 4 4096:4096:3 16384:4096:3 2>&1 | grep -v Warn
for sh in "4096 4096 2" "16384 4096 3" "28672 8192 3"; do
  echo "== trace $sh"; SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn | head -9
done
timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1
