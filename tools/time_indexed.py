"""us per GEMV of indexed-meta weights (1 B/group + table) vs the 5 B/group format, same shapes (graph ring > L2)."""
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
for name, M, N in (("q_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("down_proj", 4096, 14336)):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=1)
    table = np.stack([ri.ravel()[:256], s16.ravel()[:256], b16.ravel()[:256]], 1).astype(np.int64)
    idx = np.random.default_rng(0).integers(0, 256, size=(M, N // 128)).astype(np.uint8)
    for kind in ("group", "indexed"):
        w0 = sb.pack_canonical(pc, s16, b16, ri, 16, device=dev) if kind == "group" else sb.pack_indexed(pc, idx, table, device=dev)
        ring = bench._ring_count(w0.nbytes)
        ws_ = [w0] + [sb.SbvrWeights(M, N, 4, 16, w0.data.clone(), w0.ratio_pow.clone(), w0.meta_kind, w0.coef_table)
                      for _ in range(ring - 1)]
        wsp = [sb.Workspace.for_weights(w, 1) for w in ws_]
        act = sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=6)).to(dev))
        y = torch.empty(1, M, device=dev)
        med, p10, p90 = bench._graph_stats(torch.cuda.Stream(dev), lambda i: sb.gemv_ex(ws_[i % ring], act, y=y, ws=wsp[i % ring]), 100)
        orig = sb.algorithmic_bytes(M, N, 4)
        print(json.dumps({"shape": name, "meta": kind, "bytes": int(w0.nbytes), "us_median": round(med, 3),
                          "GBps_own_bytes": round(w0.nbytes / med / 1e3, 1),
                          "GBps_of_5B_format_bytes": round(orig / med / 1e3, 1)}), flush=True)
        del ws_, wsp
        torch.cuda.empty_cache()
