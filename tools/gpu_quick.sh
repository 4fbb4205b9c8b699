#!/bin/bash
# Quick GPU iteration: GPU tests (optionally a -k filter), then the default bench line.
mkdir -p gpurun_out
K=${1:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -q -m gpu -x -k "$K" > gpurun_out/gpu_tests.log 2>&1
else
  timeout 900 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests.log 2>&1
fi
echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -c 600 gpurun_out/bench.err
python - <<'P'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print({k: d.get(k) for k in ("value", "ms_per_step", "step_us", "roofline", "e2e", "clocks", "self_check")})
    print(d.get("per_gemv"))
    print(d.get("us_per_gemv_standalone"))
except Exception as e:
    print("no bench json", e)
P
