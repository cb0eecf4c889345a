#!/bin/bash
# Builds paper_2410_02367_b200/<name>.so with extra nvcc flags (A/B experiments).
R=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr "$@" -o $R/paper_2410_02367_b200/$name.so \
  $R/paper_2410_02367_b200/csrc/sab_prepass.cu $R/paper_2410_02367_b200/csrc/sab_attention.cu $R/paper_2410_02367_b200/csrc/sab_capi.cu
