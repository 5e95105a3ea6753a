timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2"
for v in 0 1 2 3; do
  for pdl in "" "--pdl"; do
    echo "== VARIANT=$v $pdl"
    SHIFTADD_VARIANT=$v timeout 120 python tools/time_gemv.py $pdl $SH 2>&1 | grep -v Warn
  done
done
echo "== VARIANT=2 PER_SM=2 --pdl"; SHIFTADD_VARIANT=2 SHIFTADD_PER_SM=2 timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
for v in 0 1; do echo "== loads-only VARIANT=$v"; SHIFTADD_VARIANT=$v SHIFTADD_EXP=3 timeout 120 python tools/time_gemv.py $SH 2>&1 | grep -v Warn; done
for sh in "4096 4096 2" "16384 4096 3" "28672 8192 3"; do
  echo "== trace V0 $sh"; SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn
done
