"""(Needs the diagnostic build: `bash tools/build_var.sh diag -DSBVR_DIAG`, run with SBVR_LIB_AB=ab/libsbvr_diag.so.)
Per-warp globaltimer stamps of the grouped step (sbvr_encode_vector + one sbvr_gemv_group over the Llama-3-8B
layer set) inside a CUDA graph of 8 consecutive steps over a ring of 4 layers: 0 warp start, 1 first unit landed,
2 last unit done (incl. its band combine), 4 smid, 5 units.  Prints percentiles (us from the step's first warp start)
and the per-SM spread of the done stamps."""
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
XCONV = os.environ.get("XCONV", "launch")
if XCONV == "kernel":
    e0, acts = 0, []
    for n in bench.INPUT_N:
        acts.append(sb.fp16q_activation(x[e0:e0 + n], l=bench.L_BITS))
        e0 += n
probs = [[(w, acts[xin], torch.zeros(r1 - r0, device=dev)) for (_, M, N, r0, r1, w, ws, xin) in mats] for mats in layers]
wss = [sb.group_workspace(p) for p in probs]
bufs = [torch.zeros(400 * 8 * 16, dtype=torch.int64, device=dev) for _ in range(STEPS)]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for s in range(STEPS):
            if XCONV != "kernel":
                sb.encode_vector(x, out=act_all)
            os.environ["SBVR_TS_PTR"] = str(bufs[s].data_ptr())
            sb.gemv_group(probs[s % 4], ws=wss[s % 4])
    os.environ.pop("SBVR_TS_PTR", None)
    for _ in range(3):
        for b in bufs:
            b.zero_()
        g.replay()
    torch.cuda.synchronize()

out = {}
for S in (4, 5, 6):
    t = bufs[S].cpu().numpy().reshape(-1, 16)
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()
    prev = bufs[S - 1].cpu().numpy().reshape(-1, 16)
    prev = prev[prev[:, 0] > 0]
    pct = (0, 10, 50, 90, 100)
    d = {"prev_done_max": round(float((prev[:, 2].max() - base) / 1e3), 2)}
    for k, nm in ((0, "start"), (7, "first_landed"), (3, "wait_released"), (6, "conv_barrier"), (8, "first_x"), (1, "first_data"),
                  (2, "done")):
        col = (t[:, k][t[:, k] > 0] - base) / 1e3
        if len(col) == 0:
            continue
        d[nm] = [round(float(np.percentile(col, q)), 2) for q in pct]
    d["units_hist"] = {int(k): int(v) for k, v in zip(*np.unique(t[:, 5], return_counts=True))}
    per_sm = {}
    for row in t:
        per_sm.setdefault(int(row[4]), []).append((row[2] - base) / 1e3)
    sm_max = np.array([max(v) for v in per_sm.values()])
    sm_min = np.array([min(v) for v in per_sm.values()])
    d["sm_done_max_pct"] = [round(float(np.percentile(sm_max, q)), 2) for q in pct]
    d["sm_internal_spread_pct"] = [round(float(np.percentile(sm_max - sm_min, q)), 2) for q in pct]
    out[f"step{S}"] = d
print(json.dumps(out, indent=1))
# systematic imbalance? done time (us from step start) by warp index in the CTA and by the CTA's rank on its SM
S = 5
t = bufs[S].cpu().numpy().reshape(-1, 16)
valid = t[:, 0] > 0
base = t[valid, 0].min()
WPC = int(os.environ.get("WPC", "16"))           # warps per CTA of the build (SBVR_GROUP_WARPS)
done = np.where(valid, (t[:, 2] - base) / 1e3, np.nan).reshape(-1, WPC)
start = np.where(valid, (t[:, 0] - base) / 1e3, np.nan).reshape(-1, WPC)
first = np.where(valid, (t[:, 1] - base) / 1e3, np.nan).reshape(-1, WPC)
print("done by warp index:", [round(float(np.nanmean(done[:, w])), 2) for w in range(WPC)])
print("loop time (done-first) by warp index:", [round(float(np.nanmean(done[:, w] - first[:, w])), 2) for w in range(WPC)])
smid = t[:, 4].reshape(-1, WPC)[:, 0]
cta_start = np.nanmin(start, axis=1)
rank = np.zeros(len(smid), int)
for sm in np.unique(smid):
    idx = np.where(smid == sm)[0]
    order = idx[np.argsort(cta_start[idx])]
    for r_, i in enumerate(order):
        rank[i] = r_
for r_ in range(int(rank.max()) + 1):
    m = rank == r_
    print(f"CTA rank {r_} on its SM: n={m.sum()} done mean {np.nanmean(done[m]):.2f} loop mean {np.nanmean((done - first)[m]):.2f}")
# within-SM: correlation of per-warp loop time with the SMSP (warp slot % 4) of its warp
print("loop time by (rank, warp%4):", {f"{r_},{s_}": round(float(np.nanmean((done - first)[rank == r_][:, s_::4])), 2)
                                         for r_ in range(int(rank.max()) + 1) for s_ in range(4)})
