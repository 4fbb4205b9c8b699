#!/bin/bash
# Iteration call: GPU parity tests, bench (no CPU baseline), ncu full capture of the GEMV kernel.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 2 -c 2 -o gpurun_out/prof_imma \
  python tools/ncu_target.py ${NCU_ARGS} > gpurun_out/ncu_full.log 2>&1
fi
