"""Row-sharded multi-GPU SBVR GEMV (north star).

Rows of W are independent and groups run along N, so splitting the output rows never cuts a
group: rank p owns rows [p*M/P, (p+1)*M/P) of every matrix, encodes and stores only its shard,
runs sbvr_gemv on it, and the full y is joined with one all-gather.  On GPUs the process group
is NCCL (NVLink 5 / NVSwitch); the same host logic runs under gloo in the CPU tests.

Nothing here touches the C-ABI directly; the per-rank compute is the library's sbvr_gemv.
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
