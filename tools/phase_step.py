"""(Needs the diagnostic build: `bash tools/build_var.sh diag -DSBVR_DIAG`, run with
SBVR_LIB_AB=ab/libsbvr_diag.so -- the production kernel has no timestamp code.)
Per-warp globaltimer stamps of the 4 GEMV launches of a bench step (qkv, o, gate_up, down) inside
a CUDA graph of 8 consecutive steps over a ring of 4 layers (as bench.py).  Env SBVR_TS_PTR gives each
launch its own stamp buffer: 0 warp start, 1 first unit landed, 2 last unit computed, 3 exit, 4 smid.
Prints, for step 5 of the graph, per launch the percentiles (us, relative to the step's first GEMV
start) and the SM-time lost between launches."""
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
bufs = [[torch.zeros(400 * 32 * 8, dtype=torch.int64, device=dev) for _ in range(4)] for _ in range(STEPS)]
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
tabs = []
for j in range(4):
    t = bufs[S][j].cpu().numpy().reshape(-1, 8)
    tabs.append(t[t[:, 0] > 0])
base = tabs[0][:, 0].min()
prev = bufs[S - 1][3].cpu().numpy().reshape(-1, 8)
prev = prev[prev[:, 0] > 0]
out = {"step_us": round(float((tabs[3][:, 3].max() - base) / 1e3), 2),
       "prev_down_exit_max": round(float((prev[:, 3].max() - base) / 1e3), 2)}
pct = (0, 10, 50, 90, 100)
for j, t in enumerate(tabs):
    name = bench.FUSED[j][0]
    d = {}
    for k, nm in enumerate(["start", "first_data", "loop_done", "exit"]):
        col = (t[:, k][t[:, k] > 0] - base) / 1e3
        d[nm] = [round(float(np.percentile(col, q)), 2) for q in pct]
    # per SM: first start and last exit of this launch
    per_sm = {}
    for row in t:
        sm = int(row[4])
        a, b = per_sm.get(sm, (1e30, 0))
        per_sm[sm] = (min(a, row[0]), max(b, row[3]))
    span = (t[:, 3].max() - t[:, 0].min()) / 1e3
    busy = np.mean([(b - a) / 1e3 for a, b in per_sm.values()])
    d["span_us"] = round(float(span), 2)
    d["mean_sm_resident_us"] = round(float(busy), 2)
    d["units_hist"] = {int(k): int(v) for k, v in zip(*np.unique(t[:, 5], return_counts=True))}
    out[name] = d
print(json.dumps(out, indent=1))
# the slowest warps of each launch: [smid, units, start, first, done, exit, after_smem_atomic, owner_pull_start]
for j, t in enumerate(tabs):
    order = np.argsort(-t[:, 3])[:5]
    rel = lambda v: round(float((v - base) / 1e3), 2) if v > 0 else None
    print(bench.FUSED[j][0], [[int(t[i, 4]), int(t[i, 5]), rel(t[i, 0]), rel(t[i, 1]), rel(t[i, 2]), rel(t[i, 3]),
                               rel(t[i, 6]), rel(t[i, 7])] for i in order])
print("non-owners (slot 7 unset), slowest:")
for j, t in enumerate(tabs):
    m = t[:, 7] == 0
    tt = t[m]
    order = np.argsort(-tt[:, 3])[:6]
    rel = lambda v: round(float((v - base) / 1e3), 2) if v > 0 else None
    print(bench.FUSED[j][0], [[int(tt[i, 4]), int(tt[i, 5]), rel(tt[i, 0]), rel(tt[i, 1]), rel(tt[i, 2]), rel(tt[i, 3]),
                               rel(tt[i, 6])] for i in order])
    # per-SM first-data time vs. done time correlation
    sm_first = {}
    for row in t:
        sm = int(row[4]); sm_first.setdefault(sm, []).append(row)
    worst = sorted(sm_first.items(), key=lambda kv: -max(r[3] for r in kv[1]))[:3]
    for sm, rows in worst:
        rows = np.array(rows)
        print("  sm", sm, "start", rel(rows[:, 0].min()), "first", [rel(v) for v in sorted(rows[:, 1])[::4]],
              "done", [rel(v) for v in sorted(rows[:, 2])[::4]])
