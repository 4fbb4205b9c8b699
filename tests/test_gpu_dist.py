"""GPU checks of the row-sharded multi-GPU path with the all-gather fused into the GEMV epilogue
(sbvr_gemv_to_peers, dist.SymmRowShardedGemv; north star).  Only one GPU is available, so:
- several "peer" buffers on the one GPU: every shard's rows must land at its offset in every buffer, the rest of
  each buffer untouched, values bit-identical to the plain GEMV of the shard;
- a world-size-1 NCCL group with torch symmetric memory: SymmRowShardedGemv equals sbvr_gemv bit for bit, also
  replayed inside a CUDA graph.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import paper_2509_18172_b200 as sb
import synthetic
from paper_2509_18172_b200 import dist as sdist

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.mark.parametrize("M_full,N,world,T", [(8192, 4096, 4, 1), (28672, 4096, 8, 1), (1024, 4096, 2, 3),
                                              (4096, 14336, 8, 1)])
def test_gemv_to_peers_offsets_and_values(M_full, N, world, T):
    peers = [torch.full((T, M_full), float("nan"), device=DEV) for _ in range(3)]
    ptrs = [p.data_ptr() for p in peers]
    refs = []
    for rank in range(world):
        r0, r1 = sdist.shard_range(M_full, world, rank)
        pc, s16, b16, ri = synthetic.random_encoded(r1 - r0, N, 4, 16, seed=rank + 31)
        w = sb.pack_canonical(pc, s16, b16, ri, 16)
        act = sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=9, T=T)).to(DEV))
        sb.gemv_to_peers(w, act, ptrs, r0, M_full)
        refs.append((r0, r1, sb.gemv_ex(w, act, algo=sb.ALGO_MMA)))
    torch.cuda.synchronize()
    for p in peers:
        for r0, r1, y in refs:
            assert torch.equal(p[:, r0:r1], y)
        assert not torch.isnan(p).any()                 # every row written exactly by its shard


def test_gemv_to_peers_rejects_bad_offsets():
    pc, s16, b16, ri = synthetic.random_encoded(64, 256, 4, 16, seed=1)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    act = sb.encode_vector(torch.zeros(256, dtype=torch.float16, device=DEV))
    buf = torch.zeros(1, 100, device=DEV)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_to_peers(w, act, [buf.data_ptr()], 64, 100)      # rows [64, 128) do not fit 100
    assert e.value.status == sb.ERR_SHAPE
    with pytest.raises(sb.SbvrError):
        sb.gemv_to_peers(w, act, [], 0, 64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_symmetric_memory_world1_matches_gemv():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV, 0))
    try:
        M, N = 4096, 4096
        pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=5)
        w = sb.pack_canonical(pc, s16, b16, ri, 16)
        x = synthetic.activation(N, seed=6)
        act = sb.encode_vector(torch.from_numpy(x).to(DEV))
        g = sdist.SymmRowShardedGemv(w, M)
        y = g(act).clone()
        ref = sb.gemv(w, act)
        torch.cuda.synchronize()
        assert torch.equal(y, ref)
        z, xp, sc = oracle.encode_vector(x[0], 128, 8)
        enc = oracle.Encoded(M, N, oracle.OracleConfig(K=4), pc, s16, b16, ri, None)
        rows = np.arange(0, M, 37)
        yo = oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows)
        assert np.abs(y.cpu().numpy()[rows] - yo).max() <= 1e-3 * np.abs(yo).max()
        # inside a CUDA graph (the bench captures the step)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            g(act)
            torch.cuda.synchronize()
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=st):
                g(act)
            g.y_full.fill_(float("nan"))
            cg.replay()
        torch.cuda.synchronize()
        assert torch.equal(g.y_full[0], ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gemv_group_to_peers_offsets_and_values(world):
    """Every rank's grouped shard launch (simulated rank by rank on the one GPU) stores each problem's rows at its
    offset in every peer buffer; bit-identical to sbvr_gemv_group of the same shard problems; nothing else written."""
    mats = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
    n_peers = 3
    fulls = [[torch.full((M,), float("nan"), device=DEV) for (M, _) in mats] for _ in range(n_peers)]
    ptrs = [[fulls[j][i].data_ptr() for j in range(n_peers)] for i in range(len(mats))]
    refs = []
    for rank in range(world):
        bases, r0s, rows = sdist.group_peer_layout([M for M, _ in mats], world, rank)
        probs = []
        for i, (M, N) in enumerate(mats):
            pc, s16, b16, ri = synthetic.random_encoded(rows[i], N, 4, 16, seed=100 * rank + i)
            w = sb.pack_canonical(pc, s16, b16, ri, 16)
            act = sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=7 + i)).to(DEV))
            probs.append((w, act))
        sb.gemv_group_to_peers(probs, ptrs, r0s, [M for M, _ in mats])
        ys = sb.gemv_group([(w, a, None) for w, a in probs])
        refs.append((r0s, rows, ys))
    torch.cuda.synchronize()
    for j in range(n_peers):
        for r0s, rows, ys in refs:
            for i in range(len(mats)):
                assert torch.equal(fulls[j][i][r0s[i]:r0s[i] + rows[i]], ys[i])
        assert not any(torch.isnan(f).any() for f in fulls[j])


def test_symmetric_memory_world1_grouped_matches_group():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(DEV, 0))
    try:
        mats = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
        ws_, acts = [], []
        for i, (M, N) in enumerate(mats):
            pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=50 + i)
            ws_.append(sb.pack_canonical(pc, s16, b16, ri, 16))
            acts.append(sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=60 + i)).to(DEV)))
        g = sdist.SymmGroupRowShardedGemv(ws_, [M for M, _ in mats])
        ys = [y.clone() for y in g(acts)]
        refs = sb.gemv_group([(w, a, None) for w, a in zip(ws_, acts)])
        torch.cuda.synchronize()
        assert all(torch.equal(y, r) for y, r in zip(ys, refs))
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            g(acts)
            torch.cuda.synchronize()
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg, stream=st):
                g(acts)
            g.y_flat.fill_(float("nan"))
            cg.replay()
        torch.cuda.synchronize()
        assert all(torch.equal(y, r) for y, r in zip(g.y_full, refs))
    finally:
        dist.destroy_process_group()
