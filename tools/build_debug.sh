#!/bin/bash
# experiment build: libmpattn with MPA_DEBUG_TRACE timestamps -> /tmp/libmpattn_dbg.so
set -e
cd "$(dirname "$0")/../paper_2506_13059_b200/csrc"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -I../../include -I."
mkdir -p /tmp/dbgobj
for f in *.cu; do nvcc $F -DMPA_DEBUG_TRACE $EXTRA -c $f -o /tmp/dbgobj/${f%.cu}.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/libmpattn_dbg.so /tmp/dbgobj/*.o
