#!/bin/bash
# Build ab/libsbvr_<tag>.so from the working tree with extra nvcc flags (e.g. -DSBVR_MMA_WARPS=24).
set -e
tag=$1; shift
mkdir -p ab/$tag
objs=""
for f in paper_2509_18172_b200/csrc/*.cu; do
  b=$(basename $f)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I include -I paper_2509_18172_b200/csrc "$@" -c $f -o ab/$tag/$b.o &
  objs="$objs ab/$tag/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ab/libsbvr_$tag.so $objs
echo ab/libsbvr_$tag.so
