"""Run sbvr_prefill a few times at one shape (for ncu captures).  Usage: python tools/run_prefill_once.py M N T"""
import sys

import torch

import paper_2509_18172_b200 as sb
import synthetic

M, N, T = (int(v) for v in sys.argv[1:4])
pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=1)
w = sb.pack_canonical(pc, s16, b16, ri, 16)
X = torch.randn(T, N, device="cuda", dtype=torch.float16)
ws = sb.prefill_workspace(w, T)
Y = torch.empty(T, M, device="cuda")
for _ in range(3):
    sb.prefill(w, X, Y, ws)
torch.cuda.synchronize()
print("ok", float(Y.abs().sum()))
