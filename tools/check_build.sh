#!/bin/bash
# Bounds-checked debug build of libshiftadd (-DSHIFTADD_BOUNDS_CHECK): shared-memory accesses
# through the wrappers, bulk-copy destinations, DSMEM stores and split-K partial stores trap on
# an out-of-range address (compute-sanitizer is disabled on this GPU pool).  Writes
# paper_2406_05981_b200/libshiftadd_chk.so; tests/test_gpu_bounds_check.py runs every device
# path of tools/sanitize_driver.py against it.
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2406_05981_b200/build_chk
pids=()
for f in paper_2406_05981_b200/csrc/*.cu; do
  nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
    -DSHIFTADD_BOUNDS_CHECK -Iinclude -Ipaper_2406_05981_b200/csrc -c "$f" \
    -o paper_2406_05981_b200/build_chk/$(basename "$f" .cu).o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a paper_2406_05981_b200/build_chk/*.o \
  -o paper_2406_05981_b200/libshiftadd_chk.so
