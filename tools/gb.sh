#!/bin/bash
# Build libsbvr; only if that succeeds, run the given command on the GPU box via gpurun.
# usage: tools/gb.sh <timeout_s> '<command>' <logfile>
set -o pipefail
python paper_2509_18172_b200/build.py > /tmp/gb_build.log 2>&1 || { grep -E "error" /tmp/gb_build.log | head -5; echo BUILD FAILED; exit 1; }
timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout $1 -- "$2" > $3 2>&1
tail -2 $3
