"""Stamps of the persistent GEMV (gemv_pipe.cu, env SBVR_TS_PTR) over the 4 launches of a bench step.
Per CTA 18 warps x 8 words: consumers [start, first data, done, -, smid]; producer [start, -, -, exit,
-, ns waiting on empty stages, ns waiting on tickets, items]; flush [start, -, -, exit, -, ns in
reductions, reductions]."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
STEPS = 8
layers = bench.build_ring(sb, 4, 1, 0, dev)
xcat = np.concatenate([synthetic.activation(n, seed=900 + i)[0] for i, n in enumerate(bench.INPUT_N)])
x = torch.from_numpy(xcat).to(dev)
act_all = sb.encode_vector(x)
acts, g0 = [], 0
for n in bench.INPUT_N:
    ng = n // sb.G
    acts.append(sb.SbvrActivation(sb.ACT_SBVR, n, 1, bench.L_BITS, act_all.data[g0 * bench.L_BITS * 4:(g0 + ng) * bench.L_BITS * 4],
                                  act_all.scales[g0:g0 + ng]))
    g0 += ng
ys = [[torch.zeros(r1 - r0, device=dev) for (_, M, N, r0, r1, w, ws, xin) in mats] for mats in layers]
W = 19
bufs = [[torch.zeros(160 * W * 8, dtype=torch.int64, device=dev) for _ in range(4)] for _ in range(STEPS)]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for s in range(STEPS):
            sb.encode_vector(x, out=act_all)
            for j, (name, M, N, r0, r1, w, ws, xin) in enumerate(layers[s % 4]):
                os.environ["SBVR_TS_PTR"] = str(bufs[s][j].data_ptr())
                sb.gemv(w, acts[xin], y=ys[s % 4][j], ws=ws)
    os.environ.pop("SBVR_TS_PTR", None)
    for _ in range(3):
        for bb in bufs:
            for b in bb:
                b.zero_()
        g.replay()
    torch.cuda.synchronize()

S = 5
base = None
pct = (0, 10, 50, 90, 100)
for j in range(4):
    t = bufs[S][j].cpu().numpy().reshape(-1, W, 8)
    t = t[t[:, 0, 0] > 0]
    if base is None:
        base = t[:, :, 0][t[:, :, 0] > 0].min()
    rel = lambda a: [round(float(np.percentile((a - base) / 1e3, q)), 2) for q in pct]
    cons = t[:, :16]
    prod = t[:, 16]
    fl = t[:, 17]
    red = t[:, 18]
    out = {"gemv": bench.FUSED[j][0], "ctas": int(len(t)),
           "cta_start": rel(t[:, 0, 0]), "first_data": rel(cons[:, :, 1].ravel()), "cons_done": rel(cons[:, :, 2].ravel()),
           "prod_exit": rel(prod[:, 3]), "flush_exit": rel(fl[:, 3]),
           "prod_wait_empty_us": [round(float(np.percentile(prod[:, 5] / 1e3, q)), 2) for q in pct],
           "prod_wait_ticket_us": [round(float(np.percentile(prod[:, 6] / 1e3, q)), 2) for q in pct],
           "items": [int(np.percentile(prod[:, 7], q)) for q in pct],
           "red_exit": rel(red[:, 3]),
           "reduce_us_total": [round(float(np.percentile(red[:, 5] / 1e3, q)), 2) for q in pct],
           "reductions": [int(np.percentile(red[:, 6], q)) for q in pct]}
    print(json.dumps(out))
