timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SH="4096:4096:2 4096:4096:3 16384:4096:2 16384:4096:3 28672:8192:3 4096:11008:2"
for ur in 0 1; do echo "== UNIT_RELEASE=$ur --pdl"; SHIFTADD_UNIT_RELEASE=$ur timeout 120 python tools/time_gemv.py --pdl $SH 2>&1 | grep -v Warn; done
for ur in 0 1; do echo "== trace UR=$ur"; SHIFTADD_UNIT_RELEASE=$ur SHIFTADD_EXP=4 timeout 60 python tools/trace_gemv.py 4096 4096 2 2>&1 | grep -v Warn | head -9; done
