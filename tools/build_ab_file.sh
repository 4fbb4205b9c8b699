#!/bin/bash
# Build ab/libsbvr_<tag>.so from the working tree with gemv_mma.cu replaced by file $1.
set -e
file=$1; tag=$2
mkdir -p ab/$tag
cp $file ab/$tag/gemv_mma.cu
objs=""
for f in paper_2509_18172_b200/csrc/*.cu; do
  b=$(basename $f)
  src=$f; [ "$b" = "gemv_mma.cu" ] && src=ab/$tag/gemv_mma.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I include -I paper_2509_18172_b200/csrc -c $src -o ab/$tag/$b.o &
  objs="$objs ab/$tag/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ab/libsbvr_$tag.so $objs
echo ab/libsbvr_$tag.so
