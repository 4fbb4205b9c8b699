"""Per-shape us/GEMV of the batch-1 SBVR-x GEMV: sbvr_gemv (MMA kernel) vs a one-problem sbvr_gemv_group launch,
back-to-back launches over a ring of weight copies > L2 in one CUDA graph (bench.py's record method)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

dev = torch.device("cuda", 0)
shapes = [("k_proj", 1024, 4096), ("q_proj", 4096, 4096), ("qkv", 6144, 4096), ("gate_proj", 14336, 4096),
          ("down_proj", 4096, 14336), ("gate_up", 28672, 4096), ("70b_down", 8192, 28672), ("70b_down_p8", 1024, 28672),
          ("70b_gate_p8", 3584, 8192)]
st = torch.cuda.Stream()
for name, M, N in shapes:
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=5)
    w0 = sb.pack_canonical(pc, s16, b16, ri, 16)
    ring = bench._ring_count(w0.nbytes)
    ws_list = [w0] + [sb.SbvrWeights(M, N, 4, 16, w0.data.clone(), w0.ratio_pow.clone()) for _ in range(ring - 1)]
    x = torch.from_numpy(synthetic.activation(N, seed=6)).to(dev)
    act = sb.encode_vector(x)
    y = torch.empty(M, device=dev)
    wss = [sb.Workspace.for_weights(w, 1) for w in ws_list]
    gws = [sb.group_workspace([(w, act, y)]) for w in ws_list]
    iters = 60
    mma = bench._graph_stats(st, lambda i: sb.gemv(ws_list[i % ring], act, y=y, ws=wss[i % ring]), iters)
    grp = bench._graph_stats(st, lambda i: sb.gemv_group([(ws_list[i % ring], act, y)], ws=gws[i % ring]), iters)
    b = sb.algorithmic_bytes(M, N, 4)
    print(json.dumps({"shape": name, "M": M, "N": N, "mma_us": round(mma[0], 2), "group_us": round(grp[0], 2),
                      "group_GBps": round(b / (grp[0] * 1e-6) / 1e9, 1)}), flush=True)
    del ws_list, wss, gws
    torch.cuda.empty_cache()
