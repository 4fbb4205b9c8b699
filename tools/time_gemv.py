"""Per-shape GEMV timing: CUDA graph of back-to-back launches over a ring of distinct weight copies
(ring bytes > L2), device time by CUDA events.  Prints one JSON line per (shape, algo, T)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_18172_b200 as sb  # noqa: E402
import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="q_proj,k_proj,gate_proj,down_proj")
ap.add_argument("--K", type=int, default=4)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--algo", default="3", help="comma list: 1 popc, 2 tc, 3 mma")
ap.add_argument("--T", default="1", help="comma list of batch sizes")
ap.add_argument("--x", default="sbvr", choices=["sbvr", "fp16"], help="activation path")
a = ap.parse_args()
shapes = {n: (M, N) for n, M, N in synthetic.LLAMA3_8B_LAYER + [("70b_down", 8192, 28672), ("70b_gate", 28672, 8192)]}
for name in a.shapes.split(","):
    M, N = shapes[name]
    pc, s16, b16, ri = synthetic.random_encoded(M, N, a.K, 16, seed=5)
    w0 = sb.pack_canonical(pc, s16, b16, ri, 16)
    nb = w0.nbytes
    ring = max(2, int(4 * 132e6 // nb) + 1)
    ws_list = [w0] + [sb.SbvrWeights(M, N, a.K, 16, w0.data.clone(), w0.ratio_pow.clone()) for _ in range(ring - 1)]
    for T in [int(t) for t in a.T.split(",")]:
        x = torch.from_numpy(synthetic.activation(N, seed=6, T=T)).cuda()
        act = sb.encode_vector(x) if a.x == "sbvr" else sb.fp16_activation(x)
        wss = [sb.Workspace.for_weights(w, T) for w in ws_list]
        y = torch.empty(T, M, dtype=torch.float32, device="cuda")
        for algo in [int(v) for v in a.algo.split(",")]:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for i in range(3):
                    sb.gemv_ex(ws_list[i % ring], act, y=y, ws=wss[i % ring], algo=algo)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(a.iters):
                        sb.gemv_ex(ws_list[i % ring], act, y=y, ws=wss[i % ring], algo=algo)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                g.replay()
                e1.record(st)
                torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.iters
            byts = sb.algorithmic_bytes(M, N, a.K, act=a.x, T=T)
            print(json.dumps({"shape": name, "M": M, "N": N, "K": a.K, "algo": algo, "T": T, "x": a.x, "ring": ring,
                              "us": round(us, 3), "GBps": round(byts / (us * 1e-6) / 1e9, 1)}), flush=True)
