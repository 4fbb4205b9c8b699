#!/bin/bash
# Round-2 evidence: smoke, GPU tests, default bench, reference arm, ncu launch list / DRAM traffic of the step's GEMV
# launches / full captures of the batch-1 MMA GEMV (fused gate_up) and the tcgen05 batched GEMV (gate_proj, T=16).
mkdir -p gpurun_out
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
( time timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ) 2> gpurun_out/bench.time
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cublas --no-encode --no-sweeps > gpurun_out/bench_ncu.json 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:gemv_mma -c 8 --csv --log-file gpurun_out/traffic.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-cublas --no-encode --no-sweeps > gpurun_out/bench_traffic.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_mma -s 2 -c 1 -o /tmp/prof_gateup \
  python tools/ncu_target.py --M 28672 --N 4096 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/prof_gateup.ncu-rep --page raw --csv > gpurun_out/prof_gateup_raw.csv 2>/dev/null
ncu -i /tmp/prof_gateup.ncu-rep --page details --csv > gpurun_out/prof_gateup_details.csv 2>/dev/null
ncu -i /tmp/prof_gateup.ncu-rep --page source --csv > gpurun_out/prof_gateup_source.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_zt -s 2 -c 1 -o /tmp/prof_zt \
  python tools/ncu_target.py --M 14336 --N 4096 --T 16 --algo 5 > gpurun_out/ncu_zt.log 2>&1
ncu -i /tmp/prof_zt.ncu-rep --page details --csv > gpurun_out/prof_zt_details.csv 2>/dev/null
ncu -i /tmp/prof_zt.ncu-rep --page raw --csv > gpurun_out/prof_zt_raw.csv 2>/dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host.txt 2>&1; nproc >> gpurun_out/host.txt
du -sh gpurun_out
tail -2 gpurun_out/gpu_tests.log; cat gpurun_out/bench.time; tail -c 300 gpurun_out/bench.err
