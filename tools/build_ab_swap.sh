#!/bin/bash
# Build ab/libsbvr_<tag>.so from the working tree with csrc/<name> replaced by file <file>:
#   tools/build_ab_swap.sh <file> <name> <tag> [extra nvcc flags]
set -e
file=$1; name=$2; tag=$3; shift 3
mkdir -p ab/$tag
cp $file ab/$tag/$name
objs=""
for f in paper_2509_18172_b200/csrc/*.cu; do
  b=$(basename $f)
  src=$f; [ "$b" = "$name" ] && src=ab/$tag/$name
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I include -I paper_2509_18172_b200/csrc "$@" -c $src -o ab/$tag/$b.o &
  objs="$objs ab/$tag/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ab/libsbvr_$tag.so $objs
echo ab/libsbvr_$tag.so
