"""paper_2509_18172_b200 -- SBVR (arXiv 2509.18172) hot path on B200, Python binding.

This module only marshals arguments into the C-ABI of ``libsbvr.so`` (``include/sbvr.h``):
torch tensors provide device memory and the current CUDA stream; every step of the path
runs in the library's CUDA kernels.  There is no CPU fallback: if the shared library cannot
be loaded the import of the first call raises.

Names follow the C-ABI: ``encode_weights``, ``encode_vector``, ``gemv``, ``gemv_batched``
(plus ``gemv_ex``, ``debug_partials``, ``pack_canonical``, ``unpack_canonical``).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import build as _build

_lib = None

OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_UNSUPPORTED, ERR_ALIGNMENT, ERR_CUDA, ERR_WORKSPACE = range(7)
F32, F16, BF16 = 0, 1, 2
ACT_FP16, ACT_SBVR, ACT_FP16_Q = 0, 1, 2
ALGO_AUTO, ALGO_POPC, ALGO_TC, ALGO_MMA, ALGO_PIPE, ALGO_ZT = 0, 1, 2, 3, 4, 5
META_GROUP, META_INDEXED = 0, 1
G = 128


class SbvrError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str):
        super().__init__(f"{what} failed: status {status} ({detail})")
        self.status = status


class _EncCfg(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int32), ("group_size", ctypes.c_int32), ("n_ratio", ctypes.c_int32),
                ("n_scale", ctypes.c_int32), ("n_bias", ctypes.c_int32), ("s_min_factor", ctypes.c_double),
                ("strict", ctypes.c_int32)]


class _Weights(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("N", ctypes.c_int32), ("K", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("n_ratio", ctypes.c_int32), ("data", ctypes.c_void_p), ("ratio_pow", ctypes.c_void_p),
                ("meta_kind", ctypes.c_int32), ("coef_table", ctypes.c_void_p)]


class _Act(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("N", ctypes.c_int32), ("group_size", ctypes.c_int32),
                ("l", ctypes.c_int32), ("data", ctypes.c_void_p), ("scales", ctypes.c_void_p)]


def lib_path() -> str:
    return _build.LIB


def lib():
    """Load libsbvr.so (building it in-tree with nvcc if it is missing or stale)."""
    global _lib
    if _lib is None:
        ab = os.environ.get("SBVR_LIB_AB")          # A/B timing of an alternative build (tools/ only)
        if not ab and not _build.up_to_date():
            _build.build()
        L = ctypes.CDLL(ab or _build.LIB)
        P, i32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_size_t
        L.sbvr_abi_version.restype = i32
        L.sbvr_status_string.restype = ctypes.c_char_p
        L.sbvr_status_string.argtypes = [i32]
        L.sbvr_last_error.restype = ctypes.c_char_p
        L.sbvr_weights_bytes.argtypes = [i32, i32, i32, i32, i32, P, P]
        L.sbvr_encode_weights.argtypes = [P, P, i32, i32, i32, P, P, P]
        L.sbvr_encode_vector.argtypes = [P, i32, i32, i32, i32, P, P, P]
        L.sbvr_gemv_workspace_bytes.argtypes = [P, i32, P]
        L.sbvr_workspace_init.argtypes = [P, sz, P]
        L.sbvr_gemv.argtypes = [P, P, P, P, sz, P]
        L.sbvr_gemv_batched.argtypes = [P, P, i32, P, P, sz, P]
        L.sbvr_gemv_ex.argtypes = [P, P, i32, P, P, sz, i32, P]
        L.sbvr_debug_partials.argtypes = [P, P, i32, P, P]
        L.sbvr_pack_canonical.argtypes = [i32, i32, i32, i32, P, P, P, P, P]
        L.sbvr_unpack_canonical.argtypes = [i32, i32, i32, i32, P, P, P, P, P]
        L.sbvr_fill_ratio_table.argtypes = [P, P]
        L.sbvr_hadamard_rows.argtypes = [P, P, i32, i32, i32, i32, P, P]
        L.sbvr_encode_weights_cached.argtypes = [P, i32, ctypes.c_double, P, i32, i32, i32, P, P, P, P]
        if hasattr(L, "sbvr_debug_zt_sums"):
            L.sbvr_debug_zt_sums.argtypes = [P, P, i32, P, P]
        for name, at in (("sbvr_weights_bytes_ex", [i32, i32, i32, i32, i32, i32, P, P, P]),
                         ("sbvr_encode_weights_indexed", [P, i32, P, i32, i32, i32, P, P, P, sz, P]),
                         ("sbvr_pack_indexed", [i32, i32, i32, i32, P, P, P]),
                         ("sbvr_unpack_indexed", [i32, i32, i32, i32, P, P, P])):
            if hasattr(L, name):
                getattr(L, name).argtypes = at
        if hasattr(L, "sbvr_gemv_chain"):
            L.sbvr_gemv_chain.argtypes = [P, P, i32, P, P, sz, P, P]
        if hasattr(L, "sbvr_gemv_group"):
            L.sbvr_gemv_group.argtypes = [P, i32, P, sz, P]
            if hasattr(L, "sbvr_gemv_group_to_peers"):
                L.sbvr_gemv_group_to_peers.argtypes = [P, i32, P, i32, P, P, P, sz, P]
                L.sbvr_gemv_group_to_peers.restype = i32
            L.sbvr_gemv_group_workspace_bytes.argtypes = [P, i32, P]
        if hasattr(L, "sbvr_prefill"):
            L.sbvr_prefill.argtypes = [P, P, i32, P, P, sz, P]
            L.sbvr_prefill_workspace_bytes.argtypes = [P, i32, P]
        if hasattr(L, "sbvr_gemv_to_peers"):
            L.sbvr_gemv_to_peers.argtypes = [P, P, i32, P, i32, i32, i32, P, sz, P]
        # (A/B timing loads older builds through SBVR_LIB_AB: symbols they lack are simply not declared)
        for name in ("sbvr_weights_bytes", "sbvr_encode_weights", "sbvr_encode_vector", "sbvr_gemv_workspace_bytes",
                     "sbvr_workspace_init", "sbvr_gemv", "sbvr_gemv_batched", "sbvr_gemv_ex", "sbvr_debug_partials",
                     "sbvr_pack_canonical", "sbvr_unpack_canonical", "sbvr_fill_ratio_table", "sbvr_hadamard_rows", "sbvr_encode_weights_cached",
                     "sbvr_debug_zt_sums", "sbvr_gemv_to_peers", "sbvr_weights_bytes_ex",
                     "sbvr_encode_weights_indexed", "sbvr_pack_indexed", "sbvr_unpack_indexed", "sbvr_gemv_chain",
                     "sbvr_gemv_group", "sbvr_gemv_group_workspace_bytes", "sbvr_prefill", "sbvr_prefill_workspace_bytes"):
            if hasattr(L, name):
                getattr(L, name).restype = i32
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != OK:
        L = lib()
        raise SbvrError(status, what, f"{L.sbvr_status_string(status).decode()}: {L.sbvr_last_error().decode()}")


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _np_ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ weights
@dataclass
class SbvrWeights:
    M: int
    N: int
    K: int
    n_ratio: int
    data: torch.Tensor        # uint8, packed unit records (include/sbvr.h device layout)
    ratio_pow: torch.Tensor   # float32 [n_ratio, K]
    meta_kind: int = 0        # META_GROUP (5 B per group) or META_INDEXED (1 B index + coef_table)
    coef_table: Optional[torch.Tensor] = None   # META_INDEXED: int32 [1 + 2*256] (n, then (s16|b16<<16, r_idx))

    def desc(self) -> _Weights:
        return _Weights(self.M, self.N, self.K, G, self.n_ratio, self.data.data_ptr(), self.ratio_pow.data_ptr(),
                        self.meta_kind, self.coef_table.data_ptr() if self.coef_table is not None else 0)

    @property
    def nbytes(self) -> int:
        """Algorithmic bytes of the encoded weights (planes + 5 B/group metadata)."""
        return self.data.numel()


def weights_bytes(M: int, N: int, K: int, n_ratio: int = 16):
    out = [ctypes.c_size_t() for _ in range(2)]
    _check(lib().sbvr_weights_bytes(M, N, K, G, n_ratio, *[ctypes.byref(o) for o in out]), "sbvr_weights_bytes")
    return tuple(o.value for o in out)


def weights_bytes_ex(M: int, N: int, K: int, n_ratio: int = 16, meta_kind: int = META_GROUP):
    out = [ctypes.c_size_t() for _ in range(3)]
    _check(lib().sbvr_weights_bytes_ex(M, N, K, G, n_ratio, meta_kind, *[ctypes.byref(o) for o in out]),
           "sbvr_weights_bytes_ex")
    return tuple(o.value for o in out)


def weights_empty_indexed(M: int, N: int, K: int, n_ratio: int = 16, device="cuda") -> SbvrWeights:
    db, rpb, tb = weights_bytes_ex(M, N, K, n_ratio, META_INDEXED)
    dev = torch.device(device)
    return SbvrWeights(M, N, K, n_ratio, torch.empty(db, dtype=torch.uint8, device=dev),
                       torch.empty((n_ratio, K), dtype=torch.float32, device=dev), META_INDEXED,
                       torch.zeros(tb // 4, dtype=torch.int32, device=dev))


def encode_weights_indexed(W: torch.Tensor, K: int = 4, n_table: int = 256, n_ratio: int = 16, n_scale: int = 64,
                           n_bias: int = 16, s_min_factor: float = 2.0, out: Optional[SbvrWeights] = None):
    """sbvr_encode_weights_indexed (reading A23): coefficient table + a u8 index per group.
    Returns (weights, group MSE [M, N/G] fp64)."""
    assert W.is_cuda and W.dim() == 2 and W.is_contiguous()
    M, N = W.shape
    w = out if out is not None else weights_empty_indexed(M, N, K, n_ratio, W.device)
    cfg = _EncCfg(K, G, n_ratio, n_scale, n_bias, float(s_min_factor), 1)
    mse = torch.empty((M, N // G), dtype=torch.float64, device=W.device)
    scratch = torch.empty(8 * n_table, dtype=torch.uint8, device=W.device)
    d = w.desc()
    _check(lib().sbvr_encode_weights_indexed(ctypes.byref(cfg), int(n_table), _ptr(W), _DT[W.dtype], M, N,
                                             ctypes.byref(d), _ptr(mse), _ptr(scratch), scratch.numel(), _stream()),
           "sbvr_encode_weights_indexed")
    return w, mse


def table_entries(w: SbvrWeights) -> np.ndarray:
    """The coefficient table of indexed weights as [n][3] (r_idx, s16, b16) int64 (host copy)."""
    t = w.coef_table.cpu().numpy().view(np.uint32)
    n = int(t[0])
    e = t[1:1 + 2 * n].reshape(n, 2)
    return np.stack([e[:, 1], e[:, 0] & 0xFFFF, e[:, 0] >> 16], 1).astype(np.int64)


def pack_indexed(planes_canon: np.ndarray, idx: np.ndarray, table: np.ndarray, n_ratio: int = 16,
                 device="cuda") -> SbvrWeights:
    """Canonical planes + u8 table index + table [n][3] (r_idx, s16, b16) -> device indexed SbvrWeights."""
    M, NG, K, _ = planes_canon.shape
    db, _, tb = weights_bytes_ex(M, NG * G, K, n_ratio, META_INDEXED)
    data = np.zeros(db, np.uint8)
    _check(lib().sbvr_pack_indexed(M, NG * G, K, G, _np_ptr(np.ascontiguousarray(planes_canon, np.uint32)),
                                   _np_ptr(np.ascontiguousarray(idx, np.uint8)), _np_ptr(data)), "sbvr_pack_indexed")
    tab = np.zeros(tb // 4, np.uint32)
    table = np.asarray(table, np.int64).reshape(-1, 3)
    tab[0] = len(table)
    tab[1:1 + 2 * len(table):2] = (table[:, 1] | (table[:, 2] << 16)).astype(np.uint32)
    tab[2:2 + 2 * len(table):2] = table[:, 0].astype(np.uint32)
    w = weights_empty_indexed(M, NG * G, K, n_ratio, device)
    w.data.copy_(torch.from_numpy(data))
    w.coef_table.copy_(torch.from_numpy(tab.view(np.int32)))
    d = w.desc()
    _check(lib().sbvr_fill_ratio_table(ctypes.byref(d), _stream()), "sbvr_fill_ratio_table")
    return w


def unpack_indexed(w: SbvrWeights):
    """Device indexed SbvrWeights -> canonical planes [M][N/G][K][4] uint32 and index [M][N/G] uint8."""
    NG = w.N // G
    pc = np.zeros((w.M, NG, w.K, 4), np.uint32)
    idx = np.zeros((w.M, NG), np.uint8)
    data = np.ascontiguousarray(w.data.cpu().numpy(), np.uint8)
    _check(lib().sbvr_unpack_indexed(w.M, w.N, w.K, G, _np_ptr(data), _np_ptr(pc), _np_ptr(idx)), "sbvr_unpack_indexed")
    return pc, idx


def weights_empty(M: int, N: int, K: int, n_ratio: int = 16, device="cuda") -> SbvrWeights:
    db, rpb = weights_bytes(M, N, K, n_ratio)
    dev = torch.device(device)
    return SbvrWeights(M, N, K, n_ratio, torch.empty(db, dtype=torch.uint8, device=dev),
                       torch.empty((n_ratio, K), dtype=torch.float32, device=dev))


_DT = {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}


def encode_weights(W: torch.Tensor, K: int = 4, n_ratio: int = 16, n_scale: int = 64, n_bias: int = 16,
                   s_min_factor: float = 2.0, return_mse: bool = False, out: Optional[SbvrWeights] = None,
                   strict: bool = True):
    """sbvr_encode_weights: W is a CUDA [M, N] fp32/fp16/bf16 tensor.  strict=False: the fast search
    (fp32 scan, fp64 re-evaluation of the near-best entries; include/sbvr.h)."""
    assert W.is_cuda and W.dim() == 2 and W.is_contiguous()
    M, N = W.shape
    w = out if out is not None else weights_empty(M, N, K, n_ratio, W.device)
    cfg = _EncCfg(K, G, n_ratio, n_scale, n_bias, float(s_min_factor), 1 if strict else 0)
    mse = torch.empty((M, N // G), dtype=torch.float64, device=W.device) if return_mse else None
    d = w.desc()
    _check(lib().sbvr_encode_weights(ctypes.byref(cfg), _ptr(W), _DT[W.dtype], M, N, ctypes.byref(d), _ptr(mse),
                                     _stream()), "sbvr_encode_weights")
    return (w, mse) if return_mse else w


def encode_weights_cached(W: torch.Tensor, K: int = 4, cache_size: int = 8, ema_alpha: float = 0.1, n_ratio: int = 16,
                          n_scale: int = 64, n_bias: int = 16, s_min_factor: float = 2.0,
                          out: Optional[SbvrWeights] = None, strict: bool = True):
    """sbvr_encode_weights_cached: the encode-time coefficient cache (strict only).  Returns (weights,
    group MSE [M, N/G] fp64, hit [M, N/G] uint8)."""
    assert W.is_cuda and W.dim() == 2 and W.is_contiguous()
    M, N = W.shape
    w = out if out is not None else weights_empty(M, N, K, n_ratio, W.device)
    cfg = _EncCfg(K, G, n_ratio, n_scale, n_bias, float(s_min_factor), 1 if strict else 0)
    mse = torch.empty((M, N // G), dtype=torch.float64, device=W.device)
    hit = torch.empty((M, N // G), dtype=torch.uint8, device=W.device)
    d = w.desc()
    _check(lib().sbvr_encode_weights_cached(ctypes.byref(cfg), int(cache_size), float(ema_alpha), _ptr(W), _DT[W.dtype],
                                            M, N, ctypes.byref(d), _ptr(mse), _ptr(hit), _stream()),
           "sbvr_encode_weights_cached")
    return w, mse, hit


# ------------------------------------------------------------------ activations
@dataclass
class SbvrActivation:
    """An activation descriptor: SBVR-x (planes [T][N/G][l][4] + scales [T][N/G]) or fp16-x."""
    kind: int
    N: int
    T: int
    l: int
    data: torch.Tensor
    scales: Optional[torch.Tensor] = None

    def desc(self) -> _Act:
        return _Act(self.kind, self.N, G, self.l, self.data.data_ptr(),
                    self.scales.data_ptr() if self.scales is not None else 0)


def encode_vector(x: torch.Tensor, l: int = 8, out: Optional[SbvrActivation] = None) -> SbvrActivation:
    """sbvr_encode_vector: x CUDA fp16 [N] or [T, N] (Eq. 12)."""
    assert x.is_cuda and x.dtype == torch.float16 and x.is_contiguous()
    x2 = x.view(1, -1) if x.dim() == 1 else x
    T, N = x2.shape
    if out is None:
        out = SbvrActivation(ACT_SBVR, N, T, l, torch.empty(T * (N // G) * l * 4, dtype=torch.int32, device=x.device),
                             torch.empty(T * (N // G), dtype=torch.float32, device=x.device))
    _check(lib().sbvr_encode_vector(_ptr(x2), T, N, G, l, _ptr(out.data), _ptr(out.scales), _stream()),
           "sbvr_encode_vector")
    return out


def fp16q_activation(x: torch.Tensor, l: int = 8) -> SbvrActivation:
    """An fp16 activation the GEMV converts to SBVR-x itself (Eq. 12 in the kernel prologue, bit-identical to
    encode_vector; batch 1)."""
    assert x.is_cuda and x.dtype == torch.float16 and x.is_contiguous()
    x2 = x.view(1, -1) if x.dim() == 1 else x
    assert x2.shape[0] == 1
    return SbvrActivation(ACT_FP16_Q, x2.shape[1], 1, l, x2)


def fp16_activation(x: torch.Tensor) -> SbvrActivation:
    assert x.is_cuda and x.dtype == torch.float16 and x.is_contiguous()
    x2 = x.view(1, -1) if x.dim() == 1 else x
    return SbvrActivation(ACT_FP16, x2.shape[1], x2.shape[0], 0, x2)


# ------------------------------------------------------------------ GEMV
class Workspace:
    """Caller-owned GEMV workspace, initialised once by sbvr_workspace_init (kernels leave it in that
    state: publish slots re-armed, flags cleared)."""

    def __init__(self, nbytes: int, device="cuda"):
        self.nbytes = max(int(nbytes), 256)
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        _check(lib().sbvr_workspace_init(_ptr(self.buf), self.nbytes, _stream()), "sbvr_workspace_init")

    @staticmethod
    def for_weights(w: SbvrWeights, T: int = 16) -> "Workspace":
        n = ctypes.c_size_t()
        d = w.desc()
        _check(lib().sbvr_gemv_workspace_bytes(ctypes.byref(d), T, ctypes.byref(n)), "sbvr_gemv_workspace_bytes")
        return Workspace(n.value, w.data.device)


def gemv_ex(w: SbvrWeights, x: SbvrActivation, y: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None,
            algo: int = ALGO_AUTO) -> torch.Tensor:
    T = x.T
    if y is None:
        y = torch.empty((T, w.M), dtype=torch.float32, device=w.data.device)
    if ws is None:
        ws = Workspace.for_weights(w, T)
    wd, xd = w.desc(), x.desc()
    _check(lib().sbvr_gemv_ex(ctypes.byref(wd), ctypes.byref(xd), T, _ptr(y), _ptr(ws.buf), ws.nbytes, algo,
                              _stream()), "sbvr_gemv_ex")
    return y


def gemv(w: SbvrWeights, x: SbvrActivation, y: Optional[torch.Tensor] = None,
         ws: Optional[Workspace] = None) -> torch.Tensor:
    """sbvr_gemv: y[M] = W x on the SBVR weights, x SBVR-encoded or fp16."""
    assert x.T == 1
    if y is None:
        y = torch.empty(w.M, dtype=torch.float32, device=w.data.device)
    if ws is None:
        ws = Workspace.for_weights(w, 1)
    wd, xd = w.desc(), x.desc()
    _check(lib().sbvr_gemv(ctypes.byref(wd), ctypes.byref(xd), _ptr(y), _ptr(ws.buf), ws.nbytes, _stream()),
           "sbvr_gemv")
    return y


def gemv_chain(w: SbvrWeights, x: SbvrActivation, next_w: Optional[SbvrWeights], y: Optional[torch.Tensor] = None,
               ws: Optional[Workspace] = None) -> torch.Tensor:
    """sbvr_gemv_chain: as gemv/gemv_batched, plus the L2-prefetch hint for the GEMV over next_w launched next."""
    T = x.T
    if y is None:
        y = torch.empty((T, w.M) if T > 1 else (w.M,), dtype=torch.float32, device=w.data.device)
    if ws is None:
        ws = Workspace.for_weights(w, T)
    wd, xd = w.desc(), x.desc()
    nd = next_w.desc() if next_w is not None else None
    _check(lib().sbvr_gemv_chain(ctypes.byref(wd), ctypes.byref(xd), T, _ptr(y), _ptr(ws.buf), ws.nbytes,
                                 ctypes.byref(nd) if nd is not None else None, _stream()), "sbvr_gemv_chain")
    return y


def gemv_batched(w: SbvrWeights, X: SbvrActivation, Y: Optional[torch.Tensor] = None,
                 ws: Optional[Workspace] = None) -> torch.Tensor:
    """sbvr_gemv_batched: Y[T, M] for T <= 16 vectors sharing one weight fetch."""
    if Y is None:
        Y = torch.empty((X.T, w.M), dtype=torch.float32, device=w.data.device)
    if ws is None:
        ws = Workspace.for_weights(w, X.T)
    wd, xd = w.desc(), X.desc()
    _check(lib().sbvr_gemv_batched(ctypes.byref(wd), ctypes.byref(xd), X.T, _ptr(Y), _ptr(ws.buf), ws.nbytes,
                                   _stream()), "sbvr_gemv_batched")
    return Y


def gemv_to_peers(w: SbvrWeights, x: SbvrActivation, peer_ptrs, y_row_offset: int, M_full: int,
                  ws: Optional[Workspace] = None) -> None:
    """sbvr_gemv_to_peers: this rank's row-shard GEMV whose epilogue stores y into every peer's full-y buffer
    (device pointers `peer_ptrs`, [T][M_full] fp32 each) at rows [y_row_offset, y_row_offset + w.M)."""
    if ws is None:
        ws = Workspace.for_weights(w, x.T)
    arr = (ctypes.c_void_p * len(peer_ptrs))(*[int(q) for q in peer_ptrs])
    wd, xd = w.desc(), x.desc()
    _check(lib().sbvr_gemv_to_peers(ctypes.byref(wd), ctypes.byref(xd), x.T, arr, len(peer_ptrs), int(y_row_offset),
                                    int(M_full), _ptr(ws.buf), ws.nbytes, _stream()), "sbvr_gemv_to_peers")


def prefill_workspace(w: SbvrWeights, T: int) -> Workspace:
    n = ctypes.c_size_t()
    d = w.desc()
    _check(lib().sbvr_prefill_workspace_bytes(ctypes.byref(d), int(T), ctypes.byref(n)), "sbvr_prefill_workspace_bytes")
    return Workspace(n.value, w.data.device)


def prefill(w: SbvrWeights, X: torch.Tensor, Y: Optional[torch.Tensor] = None,
            ws: Optional[Workspace] = None) -> torch.Tensor:
    """sbvr_prefill (§5.1): Y[T, M] = w16 X^T with the weights decompressed to FP16 (reading A25) and the
    GEMM on tcgen05 kind::f16; X fp16 [T, N] on the device."""
    assert X.is_cuda and X.dtype == torch.float16 and X.is_contiguous()
    X2 = X.view(1, -1) if X.dim() == 1 else X
    T = X2.shape[0]
    assert X2.shape[1] == w.N
    if Y is None:
        Y = torch.empty((T, w.M), dtype=torch.float32, device=w.data.device)
    if ws is None:
        ws = prefill_workspace(w, T)
    wd = w.desc()
    _check(lib().sbvr_prefill(ctypes.byref(wd), _ptr(X2), T, _ptr(Y), _ptr(ws.buf), ws.nbytes, _stream()),
           "sbvr_prefill")
    return Y


GROUP_MAX = 8


class _Problem(ctypes.Structure):
    _fields_ = [("w", _Weights), ("x", _Act), ("y", ctypes.c_void_p)]


def _problems(problems):
    arr = (_Problem * len(problems))()
    for i, (w, x, y) in enumerate(problems):
        arr[i].w = w.desc()
        arr[i].x = x.desc()
        arr[i].y = y.data_ptr() if y is not None else 0
    return arr


def group_workspace(problems) -> Workspace:
    """Workspace for sbvr_gemv_group over `problems` [(w, x, y), ...] (y may be None here)."""
    n = ctypes.c_size_t()
    arr = _problems(problems)
    _check(lib().sbvr_gemv_group_workspace_bytes(arr, len(problems), ctypes.byref(n)), "sbvr_gemv_group_workspace_bytes")
    return Workspace(n.value, problems[0][0].data.device)


def gemv_group(problems, ws: Optional[Workspace] = None):
    """sbvr_gemv_group: independent batch-1 SBVR-x GEMVs y_p = W_p x_p in one persistent launch.
    problems: [(w, x, y or None), ...]; returns the list of y tensors."""
    problems = [(w, x, y if y is not None else torch.empty(w.M, dtype=torch.float32, device=w.data.device))
                for (w, x, y) in problems]
    if ws is None:
        ws = group_workspace(problems)
    arr = _problems(problems)
    _check(lib().sbvr_gemv_group(arr, len(problems), _ptr(ws.buf), ws.nbytes, _stream()), "sbvr_gemv_group")
    return [y for (_, _, y) in problems]


def gemv_group_to_peers(problems, peer_ptrs, y_row_offsets, M_fulls, ws: Optional[Workspace] = None) -> None:
    """sbvr_gemv_group_to_peers: this rank's row-shard problems [(w, x), ...] in one grouped launch whose epilogue
    stores problem i's y rows into every peer's full y of problem i (device pointers peer_ptrs[i][j], [M_fulls[i]]
    fp32 each) at rows [y_row_offsets[i], + w.M)."""
    n, n_peers = len(problems), len(peer_ptrs[0])
    full = [(w, x, None) for (w, x) in problems]
    if ws is None:
        ws = group_workspace(full)
    arr = _problems(full)
    ptrs = (ctypes.c_void_p * (n * n_peers))(*[int(q) for row in peer_ptrs for q in row])
    offs = (ctypes.c_int32 * n)(*[int(v) for v in y_row_offsets])
    mf = (ctypes.c_int32 * n)(*[int(v) for v in M_fulls])
    _check(lib().sbvr_gemv_group_to_peers(arr, n, ptrs, n_peers, offs, mf, _ptr(ws.buf), ws.nbytes, _stream()),
           "sbvr_gemv_group_to_peers")


def debug_partials(w: SbvrWeights, x: SbvrActivation, algo: int = ALGO_TC) -> torch.Tensor:
    P = torch.full((w.M, w.N // G, w.K, x.l), -1, dtype=torch.int32, device=w.data.device)
    wd, xd = w.desc(), x.desc()
    _check(lib().sbvr_debug_partials(ctypes.byref(wd), ctypes.byref(xd), algo, _ptr(P), _stream()),
           "sbvr_debug_partials")
    return P


def debug_zt_sums(w: SbvrWeights, x: SbvrActivation) -> torch.Tensor:
    """Test-only: the exact integers T_t = sum_e beta_t[e] z_e of the tcgen05 z-column kernel, int32
    [M, N/G, K, T] (sbvr_debug_zt_sums)."""
    T = x.T
    out = torch.full((w.M, w.N // G, w.K, T), -(2 ** 31), dtype=torch.int32, device=w.data.device)
    wd, xd = w.desc(), x.desc()
    _check(lib().sbvr_debug_zt_sums(ctypes.byref(wd), ctypes.byref(xd), T, _ptr(out), _stream()), "sbvr_debug_zt_sums")
    return out


# ------------------------------------------------------------------ host layout transforms
def pack_host(planes_canon, s16, b16, r_idx) -> np.ndarray:
    """Canonical planes [M][N/G][K][4] + meta -> packed device-layout image (numpy uint8)."""
    M, NG, K, _ = planes_canon.shape
    N = NG * G
    db, _ = weights_bytes(M, N, K)
    data = np.zeros(db, np.uint8)
    _check(lib().sbvr_pack_canonical(M, N, K, G, _np_ptr(np.ascontiguousarray(planes_canon, np.uint32)),
                                     _np_ptr(np.ascontiguousarray(s16, np.uint16)),
                                     _np_ptr(np.ascontiguousarray(b16, np.uint16)),
                                     _np_ptr(np.ascontiguousarray(r_idx, np.uint8)), _np_ptr(data)),
           "sbvr_pack_canonical")
    return data


def unpack_host(M: int, N: int, K: int, data: np.ndarray):
    NG = N // G
    pc = np.zeros((M, NG, K, 4), np.uint32)
    s16 = np.zeros((M, NG), np.uint16)
    b16 = np.zeros((M, NG), np.uint16)
    ri = np.zeros((M, NG), np.uint8)
    data = np.ascontiguousarray(data, np.uint8)
    _check(lib().sbvr_unpack_canonical(M, N, K, G, _np_ptr(data), _np_ptr(pc), _np_ptr(s16), _np_ptr(b16),
                                       _np_ptr(ri)), "sbvr_unpack_canonical")
    return pc, s16, b16, ri


def pack_canonical(planes_canon: np.ndarray, s16: np.ndarray, b16: np.ndarray, r_idx: np.ndarray, n_ratio: int = 16,
                   device="cuda") -> SbvrWeights:
    """Canonical planes + meta -> device SbvrWeights (host transform, upload, ratio table)."""
    M, NG, K, _ = planes_canon.shape
    data = pack_host(planes_canon, s16, b16, r_idx)
    w = weights_empty(M, NG * G, K, n_ratio, device)
    w.data.copy_(torch.from_numpy(data))
    d = w.desc()
    _check(lib().sbvr_fill_ratio_table(ctypes.byref(d), _stream()), "sbvr_fill_ratio_table")
    return w


def unpack_canonical(w: SbvrWeights):
    """Device SbvrWeights -> canonical numpy (planes [M][N/G][K][4] uint32, s16, b16, r_idx [M][N/G])."""
    return unpack_host(w.M, w.N, w.K, w.data.cpu().numpy())


def algorithmic_bytes(M: int, N: int, K: int, act: str = "sbvr", l: int = 8, T: int = 1) -> int:
    """B = M N K/8 + 5 M N/G + x + 4 M (x = 2N fp16, or N l/8 + 4 N/G SBVR), per token for x/y."""
    x = 2 * N if act == "fp16" else N * l // 8 + 4 * (N // G)
    return M * N * K // 8 + 5 * M * (N // G) + T * (x + 4 * M)


def hadamard_rows(X: torch.Tensor, signs: torch.Tensor, block: int = 128, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """sbvr_hadamard_rows (§4.5): randomized block Hadamard rotation of every row of X (fp32 or fp16,
    [rows, N]) with the +-1 diagonal `signs` (int8 [N]); out may be X (in place)."""
    assert X.dim() == 2 and X.is_contiguous() and signs.dtype == torch.int8 and signs.numel() == X.shape[1]
    dt = {torch.float32: F32, torch.float16: F16}[X.dtype]
    if out is None:
        out = torch.empty_like(X)
    _check(lib().sbvr_hadamard_rows(_ptr(X), _ptr(out), dt, X.shape[0], X.shape[1], block, _ptr(signs), _stream()),
           "sbvr_hadamard_rows")
    return out

