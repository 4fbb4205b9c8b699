#!/bin/bash
# ablation sweep of the tensor-memory GEMV (SBVR_EXP_MODE bits, see gemv_tc.cu) + phase timestamps
for m in 0 1 2 4 6 7; do echo "mode $m"; SBVR_EXP_MODE=$m timeout 120 python tools/time_gemv.py --shapes k_proj,q_proj,gate_proj; done > gpurun_out/abl.txt 2>&1
timeout 120 python tools/phase_ts.py > gpurun_out/phase.txt 2>&1
