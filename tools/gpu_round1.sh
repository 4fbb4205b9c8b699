#!/bin/bash
# One gpurun call: smoke, bench, ncu launch list, ncu full capture of the GEMV kernel.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 1000 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cublas --no-encode > gpurun_out/bench_ncu.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_tc -s 2 -c 2 -o gpurun_out/prof_imma \
  python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
