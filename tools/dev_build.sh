#!/bin/bash
# Development build of libshiftadd with per-CTA phase tracing (SHIFTADD_DEV_TRACE):
# writes paper_2406_05981_b200/libshiftadd_dev.so; load it with SHIFTADD_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -DSHIFTADD_DEV_TRACE -Iinclude -Ipaper_2406_05981_b200/csrc \
  paper_2406_05981_b200/csrc/*.cu -o paper_2406_05981_b200/libshiftadd_dev.so
