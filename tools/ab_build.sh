#!/bin/bash
# Build ab/libsbvr_<tag>.so from git ref <ref> (or the working tree if ref is "wt") for same-box A/B timing.
# Extra args are nvcc flags (e.g. -DSBVR_DIAG).
set -e
tag=$1; ref=$2; shift 2
src=paper_2509_18172_b200/csrc
if [ "$ref" != "wt" ]; then
  rm -rf /tmp/ab_$tag && mkdir -p /tmp/ab_$tag && git archive $ref $src include | tar -x -C /tmp/ab_$tag
  root=/tmp/ab_$tag
else
  root=$(pwd)
fi
mkdir -p ab/o_$tag
export root tag
export FLAGS="$*"
ls $root/$src/*.cu | xargs -P 4 -I{} sh -c 'nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -I $root/include $FLAGS -c {} -o ab/o_$tag/$(basename {}).o 2>/tmp/ab_err_$tag_$(basename {}).log || { echo "FAILED {}"; cat /tmp/ab_err_$tag_$(basename {}).log | grep error; exit 255; }'
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o ab/libsbvr_$tag.so ab/o_$tag/*.o
rm -rf ab/o_$tag
echo ab/libsbvr_$tag.so
