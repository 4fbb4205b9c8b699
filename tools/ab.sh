#!/bin/bash
# A/B timing: current build vs ab/libsbvr_<tag>.so for each tag given, twice, interleaved.
shapes=${SHAPES:-k_proj,q_proj,gate_proj,down_proj}
for i in 1 2; do
  echo "== cur"; timeout 200 python tools/time_gemv.py --shapes $shapes --algo ${ALGO:-3} 2>&1 | cut -c1-160
  for t in "$@"; do echo "== $t"; SBVR_LIB_AB=ab/libsbvr_$t.so timeout 200 python tools/time_gemv.py --shapes $shapes --algo ${ALGO:-3} 2>&1 | cut -c1-160; done
done
