mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "PIPE or pipe or full_size" > gpurun_out/t_pipe.log 2>&1; tail -2 gpurun_out/t_pipe.log
timeout 120 python tools/phase_pipe.py > gpurun_out/phase_pipe.json 2>&1; cut -c1-400 gpurun_out/phase_pipe.json | grep -o '"gemv[^,]*\|"cons_done[^]]*\|"red_exit[^]]*\|"reduce_us_total[^]]*'
for A in 4 3; do
SBVR_FORCE_ALGO=$A timeout 400 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-cublas --no-encode --no-sweeps > gpurun_out/bench_$A.json 2> gpurun_out/bench_$A.err; tail -2 gpurun_out/bench_$A.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_$A.json').read().strip().splitlines()[-1]); print('$A', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['gemv_span_us']); print([(x['gemv'],x['us_serialized']) for x in d.get('per_gemv')]); print([(x['proj'],x['us']) for x in d.get('us_per_gemv_standalone')])"
done
