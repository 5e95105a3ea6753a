SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3"
for pw in 8 1 0; do echo "== PREWAIT=$pw --pdl"; SHIFTADD_PREWAIT=$pw timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn; done
for m in 4 5; do for sh in "4096 4096 2" "16384 4096 3"; do
  echo "== trace mode $m $sh"; SHIFTADD_EXP=$m timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn | head -7
  echo "== trace mode $m $sh pdl"; SHIFTADD_EXP=$m timeout 60 python tools/trace_gemv.py $sh --pdl 2>&1 | grep -v Warn | head -7
done; done
for sh in "4096 4096 2" "16384 4096 3"; do
  echo "== trace mode 4 prewait1 $sh pdl"; SHIFTADD_PREWAIT=1 SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh --pdl 2>&1 | grep -v Warn | head -7
done
