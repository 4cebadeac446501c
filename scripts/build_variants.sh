#!/bin/bash
# Build sweep-kernel variants (dev tool): build/variants/<name>.so
set -e
cd "$(dirname "$0")/../paper_2004_13961_b200/csrc"
OUT=../../build/variants
mkdir -p $OUT
ARCH="-gencode arch=compute_100a,code=sm_100a"
build() {
  name=$1; shift
  objs=""
  for f in lp_common line_transform operator frontend vector_ops ilu_csr ilu_box ilu_box2d ilu_box3d ilu_box3d_blk box_sweep box_sweep3d slab comm pcg; do
    nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c $f.cu -o $OUT/$name.$f.o &
    objs="$objs $OUT/$name.$f.o"
  done
  wait
  nvcc $ARCH -shared -o $OUT/$name.so $objs -cudart static -ldl
  rm -f $objs
}
build "$@"
