#!/bin/bash
# Bench-step A/B: current build vs ab/libsbvr_<tag>.so for each tag given (interleaved, twice).
mkdir -p gpurun_out
run() {
  SBVR_LIB_AB=$2 timeout 300 python bench.py --steps ${STEPS:-2000} --warmup 20 --no-cpu-baseline --no-cublas --no-encode --no-sweeps > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$1.json').read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['gemv_span_us'], [x['us'] for x in d.get('us_per_gemv_standalone')])" || tail -3 gpurun_out/ab_$1.err
}
for i in 1 2; do
  run cur ""
  for t in "$@"; do run $t ab/libsbvr_$t.so; done
done
