#!/bin/bash
# Build libcellgpu with extra defines for A/B runs:
#   tools/build_variant.sh NAME -DFOO -DBAR  ->  paper_2306_11544_b200/libcellgpu_NAME.so
# (load it with CELLGPU_LIB=paper_2306_11544_b200/libcellgpu_NAME.so)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2306_11544_b200/csrc
tmp=$(mktemp -d)
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off,-fno-builtin,-O2 --expt-relaxed-constexpr -I$root/include"
objs=""
for f in capi diffusion cells checksum divisions; do
  $NVCC $FLAGS "$@" -dc -o $tmp/$f.o $src/$f.cu &
  objs="$objs $tmp/$f.o"
done
wait
$NVCC $ARCH -shared -Xcompiler -fPIC -o $root/paper_2306_11544_b200/libcellgpu_$name.so $objs
rm -rf $tmp
echo built paper_2306_11544_b200/libcellgpu_$name.so
