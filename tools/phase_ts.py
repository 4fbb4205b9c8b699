"""Per-CTA phase timestamps of one tensor-memory GEMV launch (SBVR_EXP_MODE=8, 32 stamps per CTA):
0 start, 1 setup done (TMEM alloc, barriers, PDL wait), 2 worker group 0 done, 3 control thread done,
4 exit, 5+k control thread saw unit k's A ready (k<6), 12+i/16+i/20+i group 0 thread 0: i-th unit's
TMA landed / MMAs committed / epilogue done.  Prints percentiles over CTAs (us from earliest start)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ts = torch.zeros(4096 * 32, dtype=torch.int64, device="cuda")
os.environ["SBVR_EXP_MODE"] = os.environ.get("SBVR_EXP_MODE", "8")
os.environ["SBVR_TS_PTR"] = str(ts.data_ptr())
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

names = {0: "start", 1: "setup", 2: "grp0_done", 3: "ctl_done", 4: "exit"}
for k in range(6):
    names[5 + k] = f"A_ready{k}"
for i in range(4):
    names[12 + i] = f"g0_tma{i}"
    names[16 + i] = f"g0_mma{i}"
    names[20 + i] = f"g0_epi{i}"
for name, M, N in [("k_proj", 1024, 4096), ("gate_proj", 14336, 4096)]:
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=5)
    ws = [sb.pack_canonical(pc, s16, b16, ri, 16) for _ in range(3)]
    x = torch.from_numpy(synthetic.activation(N, seed=6)).cuda()
    act = sb.encode_vector(x)
    wsp = sb.Workspace.for_weights(ws[0], 1)
    for i in range(4):
        ts.zero_()
        sb.gemv(ws[i % 3], act, ws=wsp)
        torch.cuda.synchronize()
    t = ts.cpu().numpy().reshape(-1, 32)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    out = {"shape": name, "ctas": int(len(t))}
    for k, nm in sorted(names.items()):
        col = (t[:, k][t[:, k] > 0] - base) / 1000.0
        if len(col):
            out[nm] = [round(float(np.percentile(col, q)), 2) for q in (0, 50, 100)]
    print(json.dumps(out))
