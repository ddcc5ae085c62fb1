#!/bin/bash
# Timeline of the overlapped two-level iteration: builds libmgrit_trace.so
# (mgrit_api.cu with -DMG_TRACE, the other units as built) and runs one bench solve per config.
set -e
cd "$(dirname "$0")/.."
C=paper_1910_03726_b200/csrc
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off,-O2 \
  -I include --expt-relaxed-constexpr -DMG_TRACE -c $C/mgrit_api.cu -o /tmp/mgrit_api.trace.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a /tmp/mgrit_api.trace.o $C/sweep.cu.o $C/coarse.cu.o \
  $C/levels.cu.o $C/graph.cu.o $C/psifit.cu.o $C/bounded.cu.o -o paper_1910_03726_b200/libmgrit_trace.so
