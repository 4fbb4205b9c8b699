"""(Needs the diagnostic build: `bash tools/build_var.sh diag -DSBVR_DIAG`, run with
SBVR_LIB_AB=ab/libsbvr_diag.so -- the production kernel has no timestamp code.)
Per-warp timestamps of the batch-1 MMA GEMV inside a CUDA-graph chain (env SBVR_TS_PTR):
0 warp start, 1 first unit landed, 2 last unit computed, 3 exit (after band hand-off).
Graph of 20 launches over distinct weight copies; stamps of the 10th launch (warm, PDL-overlapped).
--xq: fp16 x converted in the GEMV prologue (SBVR_ACT_FP16_Q; stamp 1 then includes the conversion).
Prints percentiles over warps in us relative to the earliest start of that launch."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
bufs = [torch.zeros(400 * 16 * 8, dtype=torch.int64, device="cuda") for _ in range(20)]
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

for name, M, N in [("k_proj", 1024, 4096), ("q_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("down_proj", 4096, 14336)]:
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=5)
    ring = max(2, int(4 * 132e6 // (M * N // 2)) + 1)
    ws = [sb.pack_canonical(pc, s16, b16, ri, 16) for _ in range(min(ring, 20))]
    x = torch.from_numpy(synthetic.activation(N, seed=6)).cuda()
    act = sb.fp16q_activation(x[0]) if "--xq" in sys.argv else sb.encode_vector(x)
    wsp = sb.Workspace.for_weights(ws[0], 1)
    y = torch.empty(1, M, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(20):
                os.environ["SBVR_TS_PTR"] = str(bufs[i].data_ptr())
                sb.gemv_ex(ws[i % len(ws)], act, y=y, ws=wsp, algo=sb.ALGO_MMA)
        os.environ.pop("SBVR_TS_PTR", None)
        for _ in range(3):
            for b in bufs:
                b.zero_()
            g.replay()
        torch.cuda.synchronize()
    t = bufs[10].cpu().numpy().reshape(-1, 8)
    t = t[t[:, 0] > 0]
    prev = bufs[9].cpu().numpy().reshape(-1, 8)
    prev = prev[prev[:, 0] > 0]
    base = t[:, 0].min()
    out = {"shape": name, "warps": int(len(t)), "prev_exit_max": round(float((prev[:, 3].max() - base) / 1e3), 2)}
    for k, nm in enumerate(["start", "first_data", "loop_done", "exit"]):
        col = (t[:, k][t[:, k] > 0] - base) / 1e3
        out[nm] = [round(float(np.percentile(col, q)), 2) for q in (0, 10, 50, 90, 100)]
    # slowest warps: which SM, how many units, when they started / got data
    order = np.argsort(-t[:, 2])[:6]
    out["slowest"] = [[int(t[j, 4]), int(t[j, 5]), round(float((t[j, 0] - base) / 1e3), 2),
                       round(float((t[j, 1] - base) / 1e3), 2), round(float((t[j, 2] - base) / 1e3), 2)] for j in order]
    per_sm = {}
    for row in t:
        per_sm.setdefault(int(row[4]), []).append((row[2] - base) / 1e3)
    sm_done = sorted((max(v), k) for k, v in per_sm.items())
    out["sm_done_pct"] = [round(float(np.percentile([x for x, _ in sm_done], q)), 2) for q in (0, 50, 90, 100)]
    out["sm_count"] = len(per_sm)
    for k, nm in ((6, "after_smem_atomic"), (7, "after_global_atomic")):
        col = (t[:, k][t[:, k] > 0] - base) / 1e3
        if len(col):
            out[nm] = [round(float(np.percentile(col, q)), 2) for q in (0, 50, 90, 100)]
    d = (t[:, 7] - t[:, 6])[(t[:, 7] > 0) & (t[:, 6] > 0)] / 1e3
    if len(d):
        out["global_publish_us"] = [round(float(np.percentile(d, q)), 2) for q in (0, 50, 90, 100)]
    nxt = bufs[11].cpu().numpy().reshape(-1, 8)
    nxt = nxt[nxt[:, 0] > 0]
    out["next_start_min"] = round(float((nxt[:, 0].min() - base) / 1e3), 2)
    smids = t[:, 4]
    out["units_hist"] = {int(k): int(v) for k, v in zip(*np.unique(t[:, 5], return_counts=True))}
    print(json.dumps(out))
