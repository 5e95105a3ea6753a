timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SHIFTADD_DYN=1 timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2 11008:4096:3"
for d in 0 1; do echo "== DYN=$d --pdl"; SHIFTADD_DYN=$d timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn; done
for sh in "16384 4096 3" "28672 8192 3"; do
  echo "== trace DYN=1 $sh"; SHIFTADD_DYN=1 SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn | head -9
done
