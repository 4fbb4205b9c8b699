"""Row-sharded multi-GPU SBVR GEMV (north star).

Rows of W are independent and groups run along N, so splitting the output rows never cuts a
group: rank p owns rows [p*M/P, (p+1)*M/P) of every matrix, encodes and stores only its shard,
runs sbvr_gemv on it, and the full y is joined with one all-gather.  On GPUs the process group
is NCCL (NVLink 5 / NVSwitch); the same host logic runs under gloo in the CPU tests.

Two ways to join y:
- `RowShardedGemv` (+ `sbvr_row_sharded`): the local GEMV, then an NCCL all-gather of the y shards;
- `SymmGroupRowShardedGemv`: the same for several matrices in one grouped launch (a decoder layer's step);
- `SymmRowShardedGemv`: the all-gather fused into the GEMV's epilogue -- every rank's kernel stores its y rows
  directly into every rank's full-y buffer in symmetric memory (torch.distributed._symmetric_memory: the same
  allocation mapped on all GPUs of the node, reached over NVLink 5 / NVSwitch), then one signal-pad barrier
  orders those stores before y is read (sbvr_gemv_to_peers; no NCCL call on the data path).

The per-rank compute is always the library's CUDA GEMV through the C-ABI.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_range(M: int, world: int, rank: int, align: int = 16):
    """Contiguous row range of `rank`; every shard is a multiple of `align` rows (16 = one tile)."""
    if M % (world * align):
        raise ValueError(f"M={M} must be divisible by world*{align}={world * align}")
    per = M // world
    return rank * per, (rank + 1) * per


def gather_rows(y_local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather row shards (last dim) into the full output, rank order = row order."""
    world = dist.get_world_size(group)
    if world == 1:
        return y_local
    shape = list(y_local.shape)
    out_shape = shape[:-1] + [shape[-1] * world]
    if y_local.dim() == 1 and dist.get_backend(group) == "nccl":
        out = torch.empty(out_shape, dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        return out
    parts = [torch.empty_like(y_local) for _ in range(world)]
    dist.all_gather(parts, y_local.contiguous(), group=group)
    return torch.cat(parts, dim=-1)


def all_gather_rows_into(out: torch.Tensor, y_local: torch.Tensor, group=None) -> None:
    """NCCL all-gather of 1-D y shards into a preallocated full y (capturable; bench.py's N > 1 step)."""
    dist.all_gather_into_tensor(out, y_local, group=group)


class RowShardedGemv:
    """y = W x with W row-sharded across the process group.

    `local_gemv(r0, r1, x) -> y_local` computes this rank's rows (on GPUs: sbvr_gemv on the
    shard encoded by `encode_shard`); `__call__` gathers the full y on every rank."""

    def __init__(self, M: int, local_gemv: Callable, group=None):
        self.M = M
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.r0, self.r1 = shard_range(M, self.world, self.rank)
        self.local_gemv = local_gemv

    def __call__(self, x) -> torch.Tensor:
        y_local = self.local_gemv(self.r0, self.r1, x)
        return gather_rows(y_local, self.group) if self.world > 1 else y_local


def peer_row_offsets(M: int, world: int):
    """Row offset of every rank's shard in the full y (what each rank's fused epilogue writes to)."""
    return [shard_range(M, world, r)[0] for r in range(world)]


class SymmRowShardedGemv:
    """y = W x, W row-sharded over the group, the all-gather fused into the GEMV epilogue.

    A symmetric-memory buffer y_full [T][M] exists on every rank; rank p's sbvr_gemv_to_peers launch stores rows
    [r0, r1) of y into all ranks' y_full through their peer pointers, then `barrier()` (signal pads, device
    side) makes every rank's stores visible before anyone reads y_full.  Capturable in a CUDA graph."""

    def __init__(self, w_shard, M: int, T: int = 1, group=None, ws: Optional[object] = None):
        import paper_2509_18172_b200 as sb
        import torch.distributed._symmetric_memory as symm_mem
        self.sb = sb
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.M, self.T = M, T
        self.r0, self.r1 = shard_range(M, self.world, self.rank)
        assert w_shard.M == self.r1 - self.r0
        self.w = w_shard
        self.ws = ws if ws is not None else sb.Workspace.for_weights(w_shard, T)
        self.y_full = symm_mem.empty((T, M), dtype=torch.float32, device=w_shard.data.device)
        self.hdl = symm_mem.rendezvous(self.y_full, self.group)
        self.peer_ptrs = [int(p) for p in self.hdl.buffer_ptrs]
        assert len(self.peer_ptrs) == self.world

    def __call__(self, act) -> torch.Tensor:
        self.sb.gemv_to_peers(self.w, act, self.peer_ptrs, self.r0, self.M, self.ws)
        self.hdl.barrier(channel=0)
        return self.y_full if self.T > 1 else self.y_full[0]


def group_peer_layout(M_fulls, world: int, rank: int):
    """Layout of a grouped, row-sharded step: the full y of problem i lives at [base_i, base_i + M_fulls[i]) of one
    flat buffer (the same on every rank); this rank writes its shard rows [r0_i, r1_i) of problem i.
    Returns (base offsets, row offsets r0_i, shard rows r1_i - r0_i)."""
    bases, r0s, rows, off = [], [], [], 0
    for M in M_fulls:
        r0, r1 = shard_range(M, world, rank)
        bases.append(off)
        r0s.append(r0)
        rows.append(r1 - r0)
        off += M
    return bases, r0s, rows


class SymmGroupRowShardedGemv:
    """Several row-sharded GEMVs (e.g. a decoder layer's projections) as ONE grouped launch per rank whose epilogue
    stores every y row into every rank's full y: one symmetric-memory buffer holds all problems' full y's
    (group_peer_layout), rank p's sbvr_gemv_group_to_peers writes its shard rows of every problem into every rank's
    copy through the peer pointers, then one signal-pad barrier orders the stores before anyone reads them.  No NCCL
    call on the data path; capturable in a CUDA graph."""

    def __init__(self, w_shards, M_fulls, group=None, ws: Optional[object] = None):
        import paper_2509_18172_b200 as sb
        import torch.distributed._symmetric_memory as symm_mem
        self.sb = sb
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.M_fulls = list(M_fulls)
        self.bases, self.r0s, rows = group_peer_layout(self.M_fulls, self.world, self.rank)
        assert [w.M for w in w_shards] == rows
        self.w = list(w_shards)
        dev = w_shards[0].data.device
        self.y_flat = symm_mem.empty((sum(self.M_fulls),), dtype=torch.float32, device=dev)
        self.hdl = symm_mem.rendezvous(self.y_flat, self.group)
        base_ptrs = [int(q) for q in self.hdl.buffer_ptrs]
        assert len(base_ptrs) == self.world
        self.peer_ptrs = [[bp + 4 * b for bp in base_ptrs] for b in self.bases]
        self.ws = ws
        self.y_full = [self.y_flat[b:b + M] for b, M in zip(self.bases, self.M_fulls)]

    def __call__(self, acts):
        probs = list(zip(self.w, acts))
        if self.ws is None:
            self.ws = self.sb.group_workspace([(w, a, None) for w, a in probs])
        self.sb.gemv_group_to_peers(probs, self.peer_ptrs, self.r0s, self.M_fulls, self.ws)
        self.hdl.barrier(channel=0)
        return self.y_full


def encode_shard(W_full: torch.Tensor, world: int, rank: int, **kw):
    """Encode only this rank's row shard of W on the local GPU (sbvr_encode_weights)."""
    import paper_2509_18172_b200 as sb
    r0, r1 = shard_range(W_full.shape[0], world, rank)
    return sb.encode_weights(W_full[r0:r1].contiguous(), **kw)


def sbvr_row_sharded(w_shard, M: int, group=None, ws: Optional[object] = None) -> RowShardedGemv:
    """RowShardedGemv whose local compute is sbvr_gemv on an already encoded shard."""
    import paper_2509_18172_b200 as sb
    wsp = ws if ws is not None else sb.Workspace.for_weights(w_shard, 1)

    def local(r0, r1, act):
        assert w_shard.M == r1 - r0
        return sb.gemv(w_shard, act, ws=wsp)

    return RowShardedGemv(M, local, group)
