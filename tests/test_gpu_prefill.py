"""GPU parity of sbvr_prefill (include/sbvr.h; §5.1: SBVR weights decompressed into FP16 and a
GEMM on the tensor cores) against the oracle O-PF (reading A25).

  * the FP16 decompression is bit-identical to oracle.prefill_decode: unit-vector tokens make Y the decompressed
    matrix itself (a single nonzero product per output, exact in fp32), K = 1..4, tail row blocks, one and two
    passes, row groups with |c16| >= 32 (the bit-select path) mixed with the fast path inside one unit;
  * random fp16 tokens: every Y element against the fp64 GEMM of the decompressed weights, normwise and floored
    relative error <= 1e-4 (fp32 accumulation over N <= 2048 products), T from 1 to 300 (ragged N tiles, two
    passes), problems smaller than one CTA's share and row blocks split across CTAs;
  * full-size Llama-3-8B shapes at the bench's T on sampled rows (bar 1e-3), determinism, the workspace's arrival
    counters back at rest (canary after it), and the ABI's rejections.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_18172_b200 as sb
import synthetic

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = 1e-4


def _close(y, ref, tol=TOL):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    nw = err.max() / scale
    fl = (err / np.maximum(np.abs(ref), 1e-2 * scale)).max()
    assert nw <= tol and fl <= tol, (nw, fl)


def _make(M, N, K, seed, big_rows=0):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=seed)
    if big_rows:
        # a few row groups with |c_t| >= 32: they take the bit-select path, their neighbours the fast path
        rng = np.random.default_rng(seed + 7)
        s = s16.view(np.float16).copy()
        pick = rng.choice(M * (N // 128), size=big_rows, replace=False)
        s.reshape(-1)[pick] = np.float16(40.0)
        s16 = s.view(np.uint16)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    enc = oracle.Encoded(M, N, oracle.OracleConfig(K=K, n_ratio=16), pc, s16, b16, ri, None)
    return w, enc


class _CanaryWs:
    CANARY = 4096

    def __init__(self, w, T):
        n = sb.prefill_workspace(w, T).nbytes
        self.full = torch.full((n + self.CANARY,), 0x5A, dtype=torch.uint8, device=DEV)
        self.buf = self.full[:n]
        self.nbytes = n
        self.buf.fill_(0xFF)
        n_rb = (w.M + 127) // 128
        Us = n_rb * (w.N // 128)
        C = min(torch.cuda.get_device_properties(0).multi_processor_count, (Us + 7) // 8)
        NT = next(v for v in (16, 32, 64, 128, 256) if min(T, 256) <= v)
        self.rest = (n_rb + 1) * 4       # the arrival counters (partial slots and token tiles: any content at rest)

    def ok(self):
        return bool(torch.all(self.full[self.nbytes:] == 0x5A)) and bool(torch.all(self.buf[:self.rest] == 0xFF))


@pytest.mark.parametrize("K", [1, 2, 3, 4])
@pytest.mark.parametrize("M,N", [(128, 256), (208, 384)])
def test_decompression_bit_exact(K, M, N):
    w, enc = _make(M, N, K, seed=10 * K + M, big_rows=3)
    w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float32)
    X = torch.eye(N, dtype=torch.float16, device=DEV)        # token j = unit vector e_j: Y[j] = column j
    Y = sb.prefill(w, X)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy(), w16.T)


@pytest.mark.parametrize("T", [1, 5, 16, 33, 100, 256, 300])
def test_prefill_small_elementwise(T):
    shapes = [(128, 128), (384, 1024), (208, 512), (640, 2048)]
    for i, (M, N) in enumerate(shapes):
        w, enc = _make(M, N, 4, seed=100 + i + 7 * T)
        X = synthetic.activation(N, seed=200 + i, T=T)
        ws = _CanaryWs(w, T)
        Y = sb.prefill(w, torch.from_numpy(X).to(DEV), ws=ws)
        Y2 = sb.prefill(w, torch.from_numpy(X).to(DEV), ws=ws)
        torch.cuda.synchronize()
        assert ws.ok()
        assert torch.equal(Y, Y2)
        _close(Y.cpu().numpy(), oracle.prefill_rows(enc, X))


@pytest.mark.parametrize("K", [2, 3])
def test_prefill_other_k(K):
    w, enc = _make(512, 1024, K, seed=300 + K)
    X = synthetic.activation(1024, seed=310 + K, T=40)
    Y = sb.prefill(w, torch.from_numpy(X).to(DEV))
    torch.cuda.synchronize()
    _close(Y.cpu().numpy(), oracle.prefill_rows(enc, X))


def _rows(M, seed, n=48):
    r = np.random.default_rng(seed).choice(M, min(M, n), replace=False)
    edges = [0, M - 1] + [b for b in (127, 128, M // 2) if b < M]
    return np.unique(np.concatenate([r, edges])).astype(np.int32)


@pytest.mark.parametrize("name,M,N,T", [("gate_proj", 14336, 4096, 16), ("gate_proj", 14336, 4096, 256),
                                        ("q_proj", 4096, 4096, 64), ("down_proj", 4096, 14336, 128)])
def test_prefill_full_size_sampled(name, M, N, T):
    w, enc = _make(M, N, 4, seed=hash(name) % 1000 + T)
    X = synthetic.activation(N, seed=400 + T, T=T)
    ws = _CanaryWs(w, T)
    Y = sb.prefill(w, torch.from_numpy(X).to(DEV), ws=ws)
    Y2 = sb.prefill(w, torch.from_numpy(X).to(DEV), ws=ws)
    torch.cuda.synchronize()
    assert ws.ok()
    assert torch.equal(Y, Y2)
    rows = _rows(M, T)
    # N = 4096 .. 14336 fp32-accumulated products: the project bar, observed ~4e-6 normwise
    _close(Y.cpu().numpy()[:, rows], oracle.prefill_rows(enc, X, rows), tol=1e-3)


def test_prefill_graph_replay():
    w, enc = _make(1024, 2048, 4, seed=500)
    X = torch.from_numpy(synthetic.activation(2048, seed=501, T=24)).to(DEV)
    Y = torch.full((24, 1024), float("nan"), device=DEV)
    ws = sb.prefill_workspace(w, 24)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        sb.prefill(w, X, Y, ws)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            sb.prefill(w, X, Y, ws)
        Y.fill_(float("nan"))
        g.replay()
        first = Y.clone()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(first, Y)
    _close(Y.cpu().numpy(), oracle.prefill_rows(enc, X.cpu().numpy()))


def test_prefill_rejections_and_empty():
    w, _ = _make(128, 256, 4, seed=600)
    ws = sb.prefill_workspace(w, 4)
    Y = torch.empty(0, 128, device=DEV)
    assert sb.prefill(w, torch.empty(0, 256, dtype=torch.float16, device=DEV), Y, ws).numel() == 0
    pc, s16, b16, ri = synthetic.random_encoded(128, 256, 4, 16, seed=601)
    wi = sb.pack_indexed(pc, np.zeros((128, 2), np.uint8), np.array([[3, 0x2C00, 0]], np.int64), 16) \
        if hasattr(sb, "pack_indexed") else None
    if wi is not None:
        with pytest.raises(sb.SbvrError) as e:
            sb.prefill(wi, torch.zeros(2, 256, dtype=torch.float16, device=DEV), ws=ws)
        assert e.value.status == sb.ERR_UNSUPPORTED
    with pytest.raises(sb.SbvrError) as e:
        sb.prefill(w, torch.zeros(2, 256, dtype=torch.float16, device=DEV), ws=sb.Workspace(256))
    assert e.value.status == sb.ERR_WORKSPACE


@pytest.mark.parametrize("M,N", [(16, 128), (48, 128), (16, 1024), (144, 256)])
@pytest.mark.parametrize("T", [1, 3, 17])
def test_prefill_tiny_shapes(M, N, T):
    """Degenerate sizes: a single 16-row tail block, one group per row (every unit its own row block), a row block
    smaller than one CTA's share, ragged token counts."""
    w, enc = _make(M, N, 4, seed=700 + M + N + T)
    X = synthetic.activation(N, seed=701 + T, T=T)
    Y = sb.prefill(w, torch.from_numpy(X).to(DEV))
    torch.cuda.synchronize()
    _close(Y.cpu().numpy(), oracle.prefill_rows(enc, X))
