#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..." : libdtopk variant for A/B runs (DTOPK_LIB=...)
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2109_08219_b200/_lib/var
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -Xptxas -v $2 -shared -o paper_2109_08219_b200/_lib/var/lib_$1.so \
  paper_2109_08219_b200/csrc/api.cu > paper_2109_08219_b200/_lib/var/ptxas_$1.log 2>&1
