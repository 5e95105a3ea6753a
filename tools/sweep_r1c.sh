for nw in 8 16; do
for sh in "4096 4096 2" "16384 4096 3" "28672 8192 3"; do
  echo "== NW=$nw $sh"; SHIFTADD_PF=0 SHIFTADD_NW=$nw SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn
done; done
