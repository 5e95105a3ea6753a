SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2"
for pn in 32 128 500; do echo "== POLLNS=$pn --pdl"; SHIFTADD_POLLNS=$pn timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn; done
for sh in "4096 4096 2" "4096 11008 2" "28672 8192 3"; do
  echo "== trace $sh"; SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn | head -9
done
