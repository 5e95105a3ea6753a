timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3"
for cfg in "8 1 0" "8 1 4" "8 1 8" "8 1 16" "16 1 6" "8 2 6" "8 2 0"; do
  set -- $cfg
  for exp in 0 3; do
    echo "== NW=$1 PER_SM=$2 PF=$3 EXP=$exp"
    SHIFTADD_NW=$1 SHIFTADD_PER_SM=$2 SHIFTADD_PF=$3 SHIFTADD_EXP=$exp timeout 120 python tools/time_gemv.py $SH 2>&1 | grep -v Warn
  done
done
for cfg in "8 1 6" "8 1 12"; do
  set -- $cfg
  echo "== PDL NW=$1 PER_SM=$2 PF=$3"
  SHIFTADD_NW=$1 SHIFTADD_PER_SM=$2 SHIFTADD_PF=$3 timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn
done
