timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2"
for cfg in "16 1" "16 2" "24 1" "32 1"; do
  set -- $cfg
  for pdl in "" "--pdl"; do
    echo "== NW=$1 PER_SM=$2 $pdl"
    SHIFTADD_NW=$1 SHIFTADD_PER_SM=$2 timeout 120 python tools/time_gemv.py $pdl $SH 2>&1 | grep -v Warn
  done
done
echo "== loads-only NW=24"; SHIFTADD_NW=24 SHIFTADD_EXP=3 timeout 120 python tools/time_gemv.py $SH 2>&1 | grep -v Warn
for sh in "4096 4096 2" "16384 4096 3" "28672 8192 3"; do
  echo "== trace NW=16 $sh"; SHIFTADD_NW=16 SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py $sh 2>&1 | grep -v Warn
done
