mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t_zb.log 2>&1; tail -3 gpurun_out/t_zb.log
python - <<'PY'
import torch, bench, json
import paper_2509_18172_b200 as sb
d = torch.device("cuda")
for name, M, N in (("q_proj", 4096, 4096), ("gate_proj", 14336, 4096)):
    for T in (2, 3, 4, 8, 16):
        for algo in (sb.ALGO_MMA, sb.ALGO_TC):
            r = bench._time_gemv(sb, d, M, N, 4, T, "sbvr", algo, iters=40)
            print(name, T, r["algo"], r["us"], r["GBps"])
PY
