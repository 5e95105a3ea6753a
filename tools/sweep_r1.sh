set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3"
for nw in 8 16; do for psm in 1 2; do
  for exp in 0 1 2 3; do
    if [ $nw = 16 ] && [ $psm = 2 ]; then continue; fi
    echo "== NW=$nw PER_SM=$psm EXP=$exp"
    SHIFTADD_NW=$nw SHIFTADD_PER_SM=$psm SHIFTADD_EXP=$exp timeout 120 python tools/time_gemv.py $SH 2>&1 | grep -v Warn
  done
done; done
echo "== PDL NW=8"
SHIFTADD_NW=8 timeout 120 python tools/time_gemv.py --pdl $SH
