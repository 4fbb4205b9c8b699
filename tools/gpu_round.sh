#!/bin/bash
# Round evidence call: smoke, GPU tests, bench (default), reference arm, ncu launch list of a short bench,
# ncu dram bytes of one step's 4 GEMV launches, ncu full capture of the gate_up GEMV.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 400 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cublas --no-encode > gpurun_out/bench_ncu.json 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemv_mma -c 8 --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cublas --no-encode > gpurun_out/bench_traffic.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_mma -s 2 -c 1 -o gpurun_out/prof_gateup \
  python tools/ncu_target.py --M 28672 --N 4096 > gpurun_out/ncu_full.log 2>&1
# keep gpurun_out under the 64 MiB copy-back limit: export the report's raw page, drop the report
ncu -i gpurun_out/prof_gateup.ncu-rep --page raw --csv > gpurun_out/prof_gateup_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_gateup.ncu-rep --page source --csv > gpurun_out/prof_gateup_source.csv 2>/dev/null
mv gpurun_out/prof_gateup.ncu-rep /tmp/ 2>/dev/null
du -sh gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt 2>&1; nproc >> gpurun_out/host.txt
