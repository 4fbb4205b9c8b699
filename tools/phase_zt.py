"""Per-phase SM-cycle totals of the ZT kernel (-DSBVR_DIAG build, env SBVR_TS_PTR): one worker thread (warp 0)
and one MMA issuer (warp 8) per CTA; prints the median over CTAs of cycles per unit for each phase.
Worker phases: 0 B build + next loads, 1 wait for the unit's weights (TMA), 2 A expansion + STTM issue + meta,
3 wait::st + fences + arrive, 4 epilogue waits for D, 5 epilogue TMEM loads, 6 epilogue math + rest,
7 row-block flush.  Issuer: 0 wait A/B ready, 1 wait D free, 2 issue 4 MMAs + commit."""
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
ap.add_argument("--T", type=int, default=8)
a = ap.parse_args()
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
os.environ["SBVR_TS_PTR"] = str(buf.data_ptr())
os.environ["SBVR_LIB_AB"] = a.lib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

pc, s16, b16, ri = synthetic.random_encoded(a.M, a.N, 4, 16, seed=1)
w = sb.pack_canonical(pc, s16, b16, ri, 16)
act = sb.encode_vector(torch.from_numpy(synthetic.activation(a.N, seed=2, T=a.T)).cuda())
for _ in range(3):
    buf.zero_()
    sb.gemv_ex(w, act, algo=sb.ALGO_ZT)
    torch.cuda.synchronize()
ts = buf.view(148, 32).cpu().numpy().astype(np.float64)
units = (a.M // 128) * (a.N // 128) / 148
names_e = ["wait_mma(k-2)", "B_build+load_x", "wait_weights", "expand+coef", "st_wait_arrive", "-", "-", "-"]
names_p = ["-", "-", "-", "-", "wait_D", "ld+math", "loop", "flush"]
names_i = ["wait_AB", "wait_D_free", "issue_commit"]
out = {"T": a.T, "units_per_cta": round(units, 2)}
out["expand_warp_cycles_per_unit"] = {n: round(float(np.median(ts[:, i])) / units, 1) for i, n in enumerate(names_e) if n != "-"}
out["epilogue_warp_cycles_per_unit"] = {n: round(float(np.median(ts[:, 8 + i])) / units, 1) for i, n in enumerate(names_p) if n != "-"}
out["issuer_cycles_per_unit"] = {n: round(float(np.median(ts[:, 16 + i])) / units, 1) for i, n in enumerate(names_i)}
out["expand_total_per_unit"] = round(float(np.median(ts[:, :8].sum(1))) / units, 1)
print(json.dumps(out))
