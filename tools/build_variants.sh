#!/bin/bash
# Build libvoxvid_b200.so variants that differ only in the render-camera TU's
# compile flags, for on-GPU A/B timing (select with VV_LIB_PATH=...).
#   tools/build_variants.sh name1 "-DFLAG=.." name2 "-DFLAG=.." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_2202_06088_b200/csrc
make -s -C $CS
NVCC=/usr/local/cuda/bin/nvcc
BASEFLAGS=${BASEFLAGS:-}
ARCH="-gencode arch=compute_100a,code=sm_100a"
OBJ=$ROOT/paper_2202_06088_b200/_lib/obj
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  d=$ROOT/variants/$name; mkdir -p $d
  (cd $CS && $NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr $flags \
      -c -o $d/cam.o vv_launch_camera.cu 2> $d/ptxas.log) &
done
wait
for d in $ROOT/variants/*/; do
  [ -f $d/cam.o ] || continue
  $NVCC $ARCH -shared -cudart=static -o $d/libvoxvid_b200.so $OBJ/vv_api.o $OBJ/vv_launch_rays.o $d/cam.o \
      $OBJ/vv_launch_scene.o $OBJ/vv_launch_misc.o $OBJ/vv_launch_light.o $OBJ/vv_launch_multi.o $OBJ/vv_host.o
  echo "$d: $(grep -A2 'k_render_cameraILi2ELi1ELb0EN2vv6EntryN' $d/ptxas.log | grep -E 'registers|spill' | tr '\n' ' ')"
done
