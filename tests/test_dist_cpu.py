"""Row-sharded multi-GPU host logic under gloo, world_size 2, on CPU.

Each rank computes its row shard with the CPU oracle standing in for the per-rank GPU GEMV
(the sharding / gather logic is the product code in paper_2509_18172_b200/dist.py); the gathered
y must equal the unsharded oracle y bit-for-bit (rows are independent, reduction order unchanged).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_18172_b200.dist import RowShardedGemv, gather_rows, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        M, N, K = 64, 256, 4
        pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=3)
        x = synthetic.activation(N, seed=4)[0]
        z, xp, sc = oracle.encode_vector(x, 128, 8)
        xdec = oracle.x_dec_sbvr(z, sc)

        def local(r0, r1, xd):
            enc = oracle.Encoded(r1 - r0, N, oracle.OracleConfig(K=K), pc[r0:r1].copy(), s16[r0:r1].copy(),
                                 b16[r0:r1].copy(), ri[r0:r1].copy(), None)
            return torch.from_numpy(oracle.gemv_rows(enc, xd))

        y = RowShardedGemv(M, local)(xdec)
        full = oracle.gemv_rows(oracle.Encoded(M, N, oracle.OracleConfig(K=K), pc, s16, b16, ri, None), xdec)
        ok = np.array_equal(y.numpy(), full)
        # batched rows gather ([T, M_local] -> [T, M])
        t = torch.arange(2 * 8, dtype=torch.float32).view(2, 8) + 100 * rank
        g = gather_rows(t)
        ok2 = g.shape == (2, 8 * world) and torch.equal(g[:, 8 * rank:8 * (rank + 1)], t)
        q.put((rank, bool(ok), bool(ok2)))
    finally:
        dist.destroy_process_group()


def test_row_sharded_gather_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1]
    assert all(r[1] and r[2] for r in res), res


def test_shard_ranges_cover_rows():
    for M in (1024, 4096, 14336, 28672, 8192):
        for world in (1, 2, 4, 8):
            rs = [shard_range(M, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == M
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all((r1 - r0) % 16 == 0 for r0, r1 in rs)
    with pytest.raises(ValueError):
        shard_range(1000, 8, 0)


def _peer_worker(rank, world, port, shared, q):
    """Emulates the fused epilogue on CPU: every rank writes its shard's y (oracle) into ONE shared full-y
    buffer at its peer_row_offsets entry -- the addressing sbvr_gemv_to_peers uses on every peer."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        from paper_2509_18172_b200.dist import peer_row_offsets, shard_range
        M, N, K = 96, 256, 4
        pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=8)
        x = synthetic.activation(N, seed=9)[0]
        z, xp, sc = oracle.encode_vector(x, 128, 8)
        r0, r1 = shard_range(M, world, rank)
        assert peer_row_offsets(M, world)[rank] == r0
        enc = oracle.Encoded(r1 - r0, N, oracle.OracleConfig(K=K), pc[r0:r1].copy(), s16[r0:r1].copy(),
                             b16[r0:r1].copy(), ri[r0:r1].copy(), None)
        shared[r0:r1] = torch.from_numpy(oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
        dist.barrier()                                   # stands in for the signal-pad barrier
        full = oracle.gemv_rows(oracle.Encoded(M, N, oracle.OracleConfig(K=K), pc, s16, b16, ri, None),
                                oracle.x_dec_sbvr(z, sc))
        q.put((rank, bool(np.array_equal(shared.numpy(), full))))
    finally:
        dist.destroy_process_group()


def test_fused_epilogue_addressing_gloo_world3():
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    shared = torch.full((96,), float("nan"), dtype=torch.float64).share_memory_()
    q = ctx.Queue()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, shared, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1, 2] and all(r[1] for r in res), res


def _group_peer_worker(rank, world, port, shared, q):
    """The grouped fused epilogue's addressing (dist.group_peer_layout, what SymmGroupRowShardedGemv hands to
    sbvr_gemv_group_to_peers): every rank writes its shard rows of several problems into ONE shared flat buffer
    of all problems' full y's; after the barrier it must equal the unsharded oracle y of every problem."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synthetic
        from paper_2509_18172_b200.dist import group_peer_layout
        mats = [(96, 256), (48, 128), (144, 384)]
        bases, r0s, rows = group_peer_layout([M for M, _ in mats], world, rank)
        fulls = []
        for i, (M, N) in enumerate(mats):
            pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=20 + i)
            x = synthetic.activation(N, seed=30 + i)[0]
            z, xp, sc = oracle.encode_vector(x, 128, 8)
            xd = oracle.x_dec_sbvr(z, sc)
            r0, r1 = r0s[i], r0s[i] + rows[i]
            enc = oracle.Encoded(r1 - r0, N, oracle.OracleConfig(K=4), pc[r0:r1].copy(), s16[r0:r1].copy(),
                                 b16[r0:r1].copy(), ri[r0:r1].copy(), None)
            shared[bases[i] + r0:bases[i] + r1] = torch.from_numpy(oracle.gemv_rows(enc, xd))
            fulls.append(oracle.gemv_rows(oracle.Encoded(M, N, oracle.OracleConfig(K=4), pc, s16, b16, ri, None), xd))
        dist.barrier()
        ok = all(np.array_equal(shared[b:b + M].numpy(), f) for b, (M, _), f in zip(bases, mats, fulls))
        q.put((rank, bool(ok and bases == [0, 96, 144])))
    finally:
        dist.destroy_process_group()


def test_grouped_fused_epilogue_addressing_gloo_world3():
    world = 3
    port = _free_port()
    ctx = mp.get_context("spawn")
    shared = torch.full((96 + 48 + 144,), float("nan"), dtype=torch.float64).share_memory_()
    q = ctx.Queue()
    procs = [ctx.Process(target=_group_peer_worker, args=(r, world, port, shared, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r[0] for r in res) == [0, 1, 2] and all(r[1] for r in res), res
