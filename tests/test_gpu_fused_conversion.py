"""The activation conversion folded into the GEMV prologue (SBVR_ACT_FP16_Q): the kernel
converts fp16 x to SBVR-x (Eq. 12) with the same fp32 IEEE operations as sbvr_encode_vector, so y must be
bit-identical to sbvr_encode_vector + sbvr_gemv, and within the §8c.5 bar of the fp64 oracle -- at small shapes with
ragged tails, zero / outlier groups, l < 8, indexed weights, full Llama shapes and the fused all-gather epilogue."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_18172_b200 as sb
import synthetic

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _close(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    scale = max(np.abs(ref).max(), 1e-30)
    assert err.max() / scale <= 1e-3 and (err / np.maximum(np.abs(ref), 1e-2 * scale)).max() <= 1e-3


@pytest.mark.parametrize("M,N,K,l", [(16, 128, 4, 8), (208, 512, 4, 8), (336, 640, 3, 8), (1024, 512, 2, 4),
                                     (272, 256, 4, 5), (1040, 1024, 4, 8), (4096, 4096, 4, 8), (4096, 14336, 4, 8),
                                     (28672, 4096, 4, 8), (1024, 28672, 4, 8)])
def test_fused_conversion_bit_identical(M, N, K, l):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M + N + K + l)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=N + l, outliers=3)
    if N >= 512:
        x[0, 128:256] = 0                                    # an all-zero group
        x[0, 300] = 127.0
    xd = torch.from_numpy(x[0]).to(DEV)
    ref = sb.gemv_ex(w, sb.encode_vector(xd, l=l), algo=sb.ALGO_MMA)[0]   # same kernel (AUTO may pick the grouped one)
    y = sb.gemv(w, sb.fp16q_activation(xd, l=l))
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    rows = np.unique(np.concatenate([np.random.default_rng(M).choice(M, min(M, 96), replace=False), [0, M - 1]]))
    z, xp, sc = oracle.encode_vector(x[0], 128, l)
    enc = oracle.Encoded(M, N, oracle.OracleConfig(K=K), pc, s16, b16, ri, None)
    _close(y.cpu().numpy()[rows], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows))


def test_fused_conversion_indexed_and_peers():
    M, N = 2048, 4096
    pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=3)
    table = np.stack([ri.ravel()[:200], s16.ravel()[:200], b16.ravel()[:200]], 1).astype(np.int64)
    idx = np.random.default_rng(1).integers(0, 200, size=(M, N // 128)).astype(np.uint8)
    wi = sb.pack_indexed(pc, idx, table)
    xd = torch.from_numpy(synthetic.activation(N, seed=4)[0]).to(DEV)
    a = sb.gemv(wi, sb.encode_vector(xd))
    b = sb.gemv(wi, sb.fp16q_activation(xd))
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    full = torch.full((1, 2 * M), float("nan"), device=DEV)
    sb.gemv_to_peers(w, sb.fp16q_activation(xd), [full.data_ptr()], M, 2 * M)
    ref = sb.gemv_ex(w, sb.encode_vector(xd), algo=sb.ALGO_MMA)[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    assert torch.equal(full[0, M:], ref) and torch.isnan(full[0, :M]).all()


def test_fused_conversion_rejections():
    pc, s16, b16, ri = synthetic.random_encoded(32, 256, 4, 16, seed=0)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x2 = torch.zeros(2, 256, dtype=torch.float16, device=DEV)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_batched(w, sb.SbvrActivation(sb.ACT_FP16_Q, 256, 2, 8, x2))
    assert e.value.status == sb.ERR_UNSUPPORTED
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_ex(w, sb.fp16q_activation(x2[0]), algo=sb.ALGO_ZT)
    assert e.value.status == sb.ERR_UNSUPPORTED
