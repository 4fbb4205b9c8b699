"""GPU parity of the coefficient table + per-group index storage (f2; reading A23):
- the indexed encoder (sample search, table, per-group best entry, bit assignment) is bit-exact against the
  oracle: table entries, planes, indices and the fp64 group MSE;
- the GEMV on indexed weights (mma.sync kernel, batch 1, 2 and the z-column batches) matches the oracle's
  decode-then-dot of the expanded table to the §8c.5 bar, with bit-exact popcount partials, at small shapes and
  sampled rows of full Llama shapes; the meta bytes per group are 1 (plus a 2 KB table per matrix).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_18172_b200 as sb
import synthetic

pytestmark = pytest.mark.gpu
DEV = "cuda"
TOL = 1e-3


def _close(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    assert err.max() / scale <= TOL and (err / np.maximum(np.abs(ref), 1e-2 * scale)).max() <= TOL


@pytest.mark.parametrize("K,M,N,n_table", [(4, 16, 512, 8), (3, 32, 256, 16), (2, 16, 1024, 4), (4, 48, 384, 256)])
def test_indexed_encoder_bitexact(K, M, N, n_table):
    W = synthetic.with_degenerate_groups(synthetic.gaussian_weight(M, N, seed=K * 7 + M, sigma=0.02), seed=K)
    cfg = oracle.OracleConfig(K=K, n_scale=16)
    ref = oracle.encode_matrix_indexed(W, cfg, n_table)
    w, mse = sb.encode_weights_indexed(torch.from_numpy(W).to(DEV), K=K, n_table=n_table, n_scale=16)
    torch.cuda.synchronize()
    assert np.array_equal(sb.table_entries(w), ref.table)
    pc, idx = sb.unpack_indexed(w)
    assert np.array_equal(pc, ref.planes) and np.array_equal(idx, ref.idx)
    assert np.array_equal(mse.cpu().numpy(), ref.mse)


def _random_indexed(M, N, K, n_tab, seed):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=seed)
    n_tab = min(n_tab, M * (N // 128))
    rng = np.random.default_rng(seed)
    table = np.stack([ri.ravel()[:n_tab], s16.ravel()[:n_tab], b16.ravel()[:n_tab]], 1).astype(np.int64)
    idx = rng.integers(0, n_tab, size=(M, N // 128)).astype(np.uint8)
    w = sb.pack_indexed(pc, idx, table)
    enc = oracle.IndexedEncoded(M, N, oracle.OracleConfig(K=K), pc, idx, table, np.zeros((M, N // 128))).expand()
    return w, enc


@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (208, 512, 4), (336, 640, 3), (1024, 512, 2), (272, 256, 4)])
@pytest.mark.parametrize("T", [1, 2, 5, 9])
def test_indexed_gemv_matches_oracle(M, N, K, T):
    w, enc = _random_indexed(M, N, K, 200, seed=M + N + K)
    X = synthetic.activation(N, seed=T, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV))
    Y = sb.gemv_ex(w, act)
    torch.cuda.synchronize()
    for t in range(T):
        z, xp, sc = oracle.encode_vector(X[t], 128, 8)
        _close(Y.cpu().numpy()[t], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
    if T == 1:
        P = sb.debug_partials(w, act, algo=sb.ALGO_MMA)
        torch.cuda.synchronize()
        z, xp, sc = oracle.encode_vector(X[0], 128, 8)
        Pref, _ = oracle.partials_rows(enc, z, xp)
        assert np.array_equal(P.cpu().numpy(), Pref)


@pytest.mark.parametrize("name,M,N", [("q_proj", 4096, 4096), ("gate_up_fused", 28672, 4096), ("down_proj", 4096, 14336)])
def test_indexed_gemv_full_size_sampled_rows(name, M, N):
    w, enc = _random_indexed(M, N, 4, 256, seed=M ^ N)
    assert w.data.numel() == M * N // 2 + M * (N // 128)          # 1 B of meta per group
    x = synthetic.activation(N, seed=4)
    act = sb.encode_vector(torch.from_numpy(x).to(DEV))
    ws = sb.Workspace.for_weights(w, 1)
    y = sb.gemv(w, act, ws=ws)
    y2 = sb.gemv(w, act, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(y, y2)
    rows = np.unique(np.concatenate([np.random.default_rng(2).choice(M, 128, replace=False), [0, 63, 64, M - 1]]))
    z, xp, sc = oracle.encode_vector(x[0], 128, 8)
    _close(y.cpu().numpy()[rows], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows))


def test_indexed_rejections():
    w, _ = _random_indexed(32, 256, 4, 8, seed=1)
    x = torch.zeros(256, dtype=torch.float16, device=DEV)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_ex(w, sb.fp16_activation(x))
    assert e.value.status == sb.ERR_UNSUPPORTED
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_ex(w, sb.encode_vector(x), algo=sb.ALGO_ZT)
    assert e.value.status == sb.ERR_UNSUPPORTED
