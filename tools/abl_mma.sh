#!/bin/bash
# Needs the diagnostic build: bash tools/build_var.sh diag -DSBVR_DIAG; runs with SBVR_LIB_AB=ab/libsbvr_diag.so
export SBVR_LIB_AB=${SBVR_LIB_AB:-ab/libsbvr_diag.so}
# MMA GEMV ablation (SBVR_EXP_MODE bits, gemv_mma.cu): 0 full, 1 no compute, 2 no TMA, 3 neither,
# 7 neither + no band flush, 8 exit after the prologue (launch floor), 4 no band flush
for m in ${MODES:-0 1 2 3 7 8 4}; do echo "== mode$m"; SBVR_EXP_MODE=$m timeout 120 python tools/time_gemv.py --shapes ${SHAPES:-k_proj,q_proj,gate_proj,down_proj} --algo 3 2>&1 | cut -c1-160; done
