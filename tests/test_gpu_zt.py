"""GPU parity of the tcgen05 z-column kernel (ALGO_ZT: batches and prefill chunks, SURVEY §8(a) a8 and
§8(f) f1; §4.4 P:245-251 per token, P:279 tensor cores amortising the weight decoding).

- the integers T_t = sum_e beta_t[e] z_e (= sum_j alpha_j popc(beta_t & d_j)) that land in tensor memory
  are bit-exact against the oracle's element-loop T (O-P), for every token of a pass;
- y for every token within the §8c.5 bar (normwise and floored relative error <= 1e-3 vs the fp64 oracle)
  for T = 1 ... 130 (one to three weight passes, ragged last pass), K = 1..4, l in {8, 5, 2}, tail row blocks
  (M % 128 != 0), shapes spanning many CTAs (cross-CTA last-arriver reduction), full-size sampled rows;
- workspace reuse and determinism; AUTO takes ZT for T >= 12.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_18172_b200 as sb
import synthetic

pytestmark = pytest.mark.gpu
TOL = 1e-3
DEV = "cuda"


def _close(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    nw = err.max() / scale
    fl = (err / np.maximum(np.abs(ref), 1e-2 * scale)).max()
    assert nw <= TOL and fl <= TOL, (nw, fl)


def _enc(pc, s16, b16, ri, K):
    M, NG = s16.shape
    return oracle.Encoded(M, NG * 128, oracle.OracleConfig(K=K, n_ratio=16), pc, s16, b16, ri, None)


@pytest.mark.parametrize("M,N,K,T,l", [(128, 128, 4, 1, 8), (144, 256, 4, 8, 8), (256, 512, 3, 13, 8),
                                       (80, 384, 2, 16, 5), (400, 640, 4, 32, 8), (48, 256, 1, 31, 2),
                                       (1024, 1024, 4, 29, 8)])
def test_zt_sums_bitexact(M, N, K, T, l):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M + N + K + T)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=T + l, T=T, outliers=2)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV), l=l)
    S = sb.debug_zt_sums(w, act)
    torch.cuda.synchronize()
    S = S.cpu().numpy()
    enc = _enc(pc, s16, b16, ri, K)
    rows = np.unique(np.concatenate([np.random.default_rng(T).choice(M, min(M, 40), replace=False), [0, M - 1]]))
    for t in range(T):
        z, xp, sc = oracle.encode_vector(X[t], 128, l)
        _, Tref = oracle.partials_rows(enc, z, xp, l=l, rows=rows)
        assert np.array_equal(S[rows, :, :, t], Tref), t


@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (208, 512, 4), (336, 640, 3), (1024, 512, 2), (272, 256, 1),
                                   (1040, 1024, 4)])
@pytest.mark.parametrize("T", [1, 2, 3, 7, 8, 9, 16, 31, 64, 65, 130])
def test_zt_gemv_matches_oracle(M, N, K, T):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=3 * M + N + K)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=T, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV))
    ws = sb.Workspace.for_weights(w, T)
    Y = sb.gemv_ex(w, act, ws=ws, algo=sb.ALGO_ZT)
    Y2 = sb.gemv_ex(w, act, ws=ws, algo=sb.ALGO_ZT)
    torch.cuda.synchronize()
    assert torch.equal(Y, Y2)
    assert torch.all(ws.buf == 0xFF)                 # workspace back at rest (counters, slots)
    enc = _enc(pc, s16, b16, ri, K)
    Yh = Y.cpu().numpy()
    for t in sorted(set([0, T - 1, T // 2, min(T - 1, 31), min(T - 1, 32)])):
        z, xp, sc = oracle.encode_vector(X[t], 128, 8)
        _close(Yh[t], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))


@pytest.mark.parametrize("l", [8, 6, 4, 2])
def test_zt_activation_bits(l):
    M, N, K, T = 256, 384, 4, 12
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=l)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=l, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV), l=l)
    Y = sb.gemv_ex(w, act, algo=sb.ALGO_ZT)
    torch.cuda.synchronize()
    enc = _enc(pc, s16, b16, ri, K)
    for t in range(T):
        z, xp, sc = oracle.encode_vector(X[t], 128, l)
        _close(Y.cpu().numpy()[t], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))


@pytest.mark.parametrize("name,M,N", [("q_proj", 4096, 4096), ("down_proj", 4096, 14336),
                                      ("gate_up_fused", 28672, 4096), ("70b_down_shard8", 1024, 28672)])
@pytest.mark.parametrize("T", [4, 16, 64])
def test_zt_full_size_sampled_rows(name, M, N, T):
    K = 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M ^ N ^ T)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=T + 3, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV))
    Y = sb.gemv_ex(w, act, algo=sb.ALGO_AUTO if T >= 12 else sb.ALGO_ZT)
    Yz = sb.gemv_ex(w, act, algo=sb.ALGO_ZT)
    torch.cuda.synchronize()
    assert torch.equal(Y, Yz)
    rows = np.unique(np.concatenate([np.random.default_rng(T).choice(M, 64, replace=False), [0, 127, 128, M - 1]]))
    enc = _enc(pc, s16, b16, ri, K)
    Yh = Y.cpu().numpy()
    for t in (0, T // 2, T - 1):
        z, xp, sc = oracle.encode_vector(X[t], 128, 8)
        _close(Yh[t][rows], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows))


def test_zt_matches_mma_path_elementwise():
    """Same integers, different fp32 association: ZT and the mma.sync z-column path agree to fp32 rounding."""
    M, N, K, T = 2048, 4096, 4, 8
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=5)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    act = sb.encode_vector(torch.from_numpy(synthetic.activation(N, seed=6, T=T)).to(DEV))
    a = sb.gemv_ex(w, act, algo=sb.ALGO_ZT)
    b = sb.gemv_ex(w, act, algo=sb.ALGO_MMA)
    torch.cuda.synchronize()
    scale = b.abs().max().item()
    assert (a - b).abs().max().item() <= 1e-5 * scale


def test_zt_rejects_what_it_does_not_cover():
    pc, s16, b16, ri = synthetic.random_encoded(32, 256, 5, 16, seed=0)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    act = sb.encode_vector(torch.zeros(4, 256, dtype=torch.float16, device=DEV))
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_ex(w, act, algo=sb.ALGO_ZT)
    assert e.value.status == sb.ERR_UNSUPPORTED
    Y = sb.gemv_batched(w, act)                      # AUTO falls back to MMA for K = 5
    torch.cuda.synchronize()
    assert not Y.any()
