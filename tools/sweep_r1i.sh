for m in 4 5; do for sh in "4096 4096 2" "16384 4096 3"; do
  echo "== trace mode $m $sh"; SHIFTADD_EXP=$m timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn | head -9
done; done
