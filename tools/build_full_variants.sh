#!/bin/bash
# Build whole-library variants of libvoxvid_b200.so that differ in -D knobs
# (VV_CAM_TH, VV_CHUNK_W, VV_SLICE_CHUNK, VV_SLICE_WARPS, VV_SLICE_BPS,
# VV_SEG_MIN, ...), each in variants/<name>/, for on-GPU A/B timing with
# VV_LIB_PATH=variants/<name>/libvoxvid_b200.so.
#   tools/build_full_variants.sh name1 "-DVV_SLICE_CHUNK=32" name2 "-DVV_CAM_TH=4" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
BASE='-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr'
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p "$ROOT/variants/$name"
  (make -s -C "$ROOT/paper_2202_06088_b200/csrc" LIBDIR="../../variants/$name" NVFLAGS="$BASE $flags" \
      > "$ROOT/variants/$name/make.log" 2>&1 && echo "$name: ok" || echo "$name: FAILED (variants/$name/make.log)") &
done
wait
