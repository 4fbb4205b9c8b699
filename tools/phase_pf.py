"""Per-phase SM-cycle totals of the prefill kernel (-DSBVR_DIAG build, env SBVR_TS_PTR), median over CTAs, per unit.
Decompression warp 0: 0 wait record, 1 loads, 2 coefficients + HFMA2 decompression, 3 wait A slot free, 4 STTM + wait
+ arrive, 5 loop.  Epilogue warp 16: 0 D ld + stores, 1 -, 2 combine, 3 wait D.  Issuer: 0 wait D free, 1 wait A,
2 issue 8 MMAs + commits.  Producer: 0 wait stage empty, 1 issue copies, 2 loop."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ap = argparse.ArgumentParser()
ap.add_argument("--lib", required=True)
ap.add_argument("--M", type=int, default=14336)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--T", type=int, default=16)
ap.add_argument("--K", type=int, default=4)
a = ap.parse_args()
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
os.environ["SBVR_TS_PTR"] = str(buf.data_ptr())
os.environ["SBVR_LIB_AB"] = a.lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

pc, s16, b16, ri = synthetic.random_encoded(a.M, a.N, 4, 16, seed=1)
w = sb.pack_canonical(pc, s16, b16, ri, 16)
X = torch.randn(a.T, a.N, device="cuda", dtype=torch.float16)
ws = sb.prefill_workspace(w, a.T)
for _ in range(3):
    buf.zero_()
    sb.prefill(w, X, ws=ws)
    torch.cuda.synchronize()
ts = buf.view(148, 32).cpu().numpy().astype(np.float64)
units = (a.M // 128) * (a.N // 128) / 148
groups = {"deq": (0, ["wait_rec", "loads", "decompress", "wait_slot", "st_wait_arrive", "loop"]),
          "epi": (8, ["ld_store", "-", "combine", "wait_D"]),
          "issuer": (16, ["wait_Dfree", "wait_A", "issue_commit"]),
          "producer": (24, ["wait_empty", "issue", "loop"])}
out = {"T": a.T, "units_per_cta": round(units, 2)}
for k, (base, names) in groups.items():
    out[k] = {n: round(float(np.median(ts[:, base + i])) / units, 1) for i, n in enumerate(names) if n != "-"}
g = ts[:, 27:32].astype(np.float64)
live = g[:, 1] > 0
g = g[live]
t0 = g[:, 1].min()
names = ["combine_first_loads", "start", "setup_done", "loops_done", "combine_done"]
out["globaltimer_us"] = {n: [round(float(np.median(g[g[:, i] > 0, i] - t0)) / 1e3, 2) if (g[:, i] > 0).any() else None,
                             round(float((g[:, i] - t0).max()) / 1e3, 2)] for i, n in enumerate(names)}
out["ctas"] = int(live.sum())
comb = g[:, 0] > 0
if comb.any():
    out["combining_ctas"] = int(comb.sum())
    out["per_cta_us"] = {"loops_to_first_loads": round(float(np.median(g[comb, 0] - g[comb, 3])) / 1e3, 2),
                         "first_loads_to_done": round(float(np.median(g[comb, 4] - g[comb, 0])) / 1e3, 2),
                         "loops_done_of_combiners": round(float(np.median(g[comb, 3] - t0)) / 1e3, 2),
                         "loops_done_of_others": round(float(np.median(g[~comb, 3] - t0)) / 1e3, 2) if (~comb).any() else None}
print(json.dumps(out))
