#!/bin/bash
# Same-box A/B: time_gemv with each ab/libsbvr_<tag>.so, interleaved twice.  Args: shapes T tags...
shapes=$1; T=$2; shift 2
for rep in 1 2; do
  for tag in "$@"; do
    SBVR_LIB_AB=ab/libsbvr_$tag.so timeout 120 python tools/time_gemv.py --shapes $shapes --algo 3 --T $T --iters 100 | \
      python -c "import sys,json; [print('$tag', json.loads(l)['shape'], json.loads(l)['us']) for l in sys.stdin]"
  done
done
