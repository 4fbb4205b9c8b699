#!/bin/bash
# Build ab/libsbvr_<tag>.so from git ref <ref> (or the working tree if ref is "wt") for same-box A/B timing.
set -e
tag=$1; ref=$2; shift 2
src=paper_2509_18172_b200/csrc
if [ "$ref" != "wt" ]; then
  rm -rf /tmp/ab_$tag && mkdir -p /tmp/ab_$tag && git archive $ref $src include | tar -x -C /tmp/ab_$tag
  root=/tmp/ab_$tag
else
  root=.
fi
mkdir -p ab/o_$tag
for f in $root/$src/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -I $root/include "$@" -c $f -o ab/o_$tag/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ab/libsbvr_$tag.so ab/o_$tag/*.o
rm -rf ab/o_$tag
echo ab/libsbvr_$tag.so
