#!/bin/bash
# Builds a tuning variant of libdigeo_b200.so into build/variants/<name>.so
#   scripts/build_variant.sh <name> [extra nvcc flags, e.g. -DDG_TRACE_MIN_BLOCKS=4]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2603_15780_b200/csrc"
out=../../build/variants/$name.so
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -Xptxas -v "$@" \
  -shared -o $out dg_capi.cu dg_trace_kernel.cu dg_diff_kernels.cu dg_capi_diff.cu dg_capi_batch.cu dg_capi_multi.cu dg_capi_poly.cu 2> ../../build/variants/$name.log
grep -A2 "trace_fast_kernelILb1" ../../build/variants/$name.log | grep -E "registers|spill" | head -3
