"""Per-CTA phase timestamps of one GEMV launch (SBVR_EXP_MODE=8): start, first TMA landed (warp 0),
warp 0 done with units, after CTA barrier, exit.  Prints percentiles relative to the earliest start."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ts = torch.zeros(4096 * 8, dtype=torch.int64, device="cuda")
os.environ["SBVR_EXP_MODE"] = "8"
os.environ["SBVR_TS_PTR"] = str(ts.data_ptr())
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

for name, M, N in [("k_proj", 1024, 4096), ("gate_proj", 14336, 4096), ("down_proj", 4096, 14336)]:
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=5)
    ws = [sb.pack_canonical(pc, s16, b16, ri, 16) for _ in range(3)]
    x = torch.from_numpy(synthetic.activation(N, seed=6)).cuda()
    act = sb.encode_vector(x)
    wsp = sb.Workspace.for_weights(ws[0], 1)
    for i in range(4):
        ts.zero_()
        sb.gemv(ws[i % 3], act, ws=wsp)
        torch.cuda.synchronize()
    t = ts.cpu().numpy().reshape(-1, 8)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    rel = (t[:, :5] - base) / 1000.0
    out = {"shape": name, "ctas": int(len(t))}
    for k, nm in enumerate(["start", "first_tma", "warp0_done", "cta_barrier", "exit"]):
        col = rel[:, k][t[:, k] > 0]
        if len(col):
            out[nm] = [round(float(np.percentile(col, q)), 2) for q in (0, 50, 90, 100)]
    print(json.dumps(out))
