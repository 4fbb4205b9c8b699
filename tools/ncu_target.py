"""Small driver for ncu: a few launches of the SBVR GEMV at one Llama shape (default gate_proj 14336x4096)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=14336)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--algo", type=int, default=sb.ALGO_MMA)
ap.add_argument("--fp16x", action="store_true")
ap.add_argument("--T", type=int, default=1)
ap.add_argument("--xq", action="store_true", help="fp16 x converted in the GEMV prologue (SBVR_ACT_FP16_Q)")
a = ap.parse_args()
pc, s16, b16, ri = synthetic.random_encoded(a.M, a.N, a.K, 16, seed=5)
ws_list = [sb.pack_canonical(pc, s16, b16, ri, 16) for _ in range(3)]   # 3 copies: no L2 reuse across launches
x = torch.from_numpy(synthetic.activation(a.N, seed=6, T=a.T)).cuda()
act = sb.fp16_activation(x[0]) if a.fp16x else (sb.fp16q_activation(x[0]) if a.xq else sb.encode_vector(x))
ws = sb.Workspace.for_weights(ws_list[0], a.T)
y = torch.empty(a.T, a.M, dtype=torch.float32, device="cuda")
for i in range(a.iters):
    sb.gemv_ex(ws_list[i % 3], act, y=y, ws=ws, algo=a.algo)
torch.cuda.synchronize()
print("done", a.M, a.N, a.K)
