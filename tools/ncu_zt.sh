#!/bin/bash
# ncu full capture of one ZT launch (gate_proj 14336x4096, T tokens) -> raw + source CSV in gpurun_out/
T=${1:-8}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:gemv_zt -s 2 -c 1 -o /tmp/prof_zt \
  python tools/ncu_target.py --M 28672 --N 8192 --T $T --algo 5 > gpurun_out/ncu_zt.log 2>&1
ncu -i /tmp/prof_zt.ncu-rep --page raw --csv > gpurun_out/prof_zt_raw.csv 2>/dev/null
ncu -i /tmp/prof_zt.ncu-rep --page source --csv > gpurun_out/prof_zt_source.csv 2>/dev/null
ncu -i /tmp/prof_zt.ncu-rep --page details --csv > gpurun_out/prof_zt_details.csv 2>/dev/null
tail -3 gpurun_out/ncu_zt.log
