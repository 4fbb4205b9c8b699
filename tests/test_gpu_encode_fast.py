"""Fast-mode encoder (sbvr_encode_config.strict = 0): fp32 scan of Algorithm 1's search space, strict
fp64 re-evaluation of the near-best entries.  Contract, checked against the oracle group by group: the chosen
entry's fp64 MSE (oracle entry_mse) <= (1 + 1e-6) x the strict best (oracle encode, Algorithm 1); the
planes are the oracle's nearest assignment for the chosen coefficients; the reported group MSE is that fp64
MSE bit for bit.  In practice the margin makes the result identical to strict mode: checked too."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_18172_b200 as sb
import synthetic

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _fp16(h):
    return float(np.array([h], np.uint16).view(np.float16)[0])


def _check_contract(Wnp, K, cfg, w_fast, mse_fast, ref):
    pc, s16, b16, ri = sb.unpack_canonical(w_fast)
    R = oracle.ratio_set(cfg.n_ratio)
    M, NG = s16.shape
    mse_fast = mse_fast.cpu().numpy()
    for r in range(M):
        for g in range(NG):
            X = Wnp[r, 128 * g:128 * (g + 1)].astype(np.float64)
            rr, ss, bb = float(R[ri[r, g]]), _fp16(s16[r, g]), _fp16(b16[r, g])
            m = oracle.entry_mse(X, K, rr, ss, bb)
            assert m <= ref.mse[r, g] * (1 + 1e-6) + 1e-300, (r, g, m, ref.mse[r, g])
            assert mse_fast[r, g] == m
            assert np.array_equal(pc[r, g], oracle.assign(X, oracle.coefficients(rr, ss, bb, K)))


@pytest.mark.parametrize("K,dtype", [(4, torch.float32), (3, torch.float32), (2, torch.bfloat16), (4, torch.float16)])
def test_encode_fast_contract_and_equal_to_strict(K, dtype):
    M, N = 32, 256
    W = synthetic.with_degenerate_groups(synthetic.gaussian_weight(M, N, seed=10 + K, sigma=0.02), seed=K)
    Wt = torch.from_numpy(W).to(dtype)
    Wnp = Wt.float().numpy()
    cfg = oracle.OracleConfig(K=K, n_ratio=16, n_scale=64 if K == 4 else 16, n_bias=16)
    kw = dict(K=K, n_ratio=cfg.n_ratio, n_scale=cfg.n_scale, n_bias=cfg.n_bias, return_mse=True)
    wf, mf = sb.encode_weights(Wt.to(DEV), strict=False, **kw)
    ws, ms = sb.encode_weights(Wt.to(DEV), strict=True, **kw)
    torch.cuda.synchronize()
    ref = oracle.encode_matrix(Wnp, cfg)
    _check_contract(Wnp, K, cfg, wf, mf, ref)
    assert torch.equal(wf.data, ws.data) and torch.equal(mf, ms)


def test_encode_fast_full_layer_equal_to_strict():
    """A 1024 x 4096 Llama-like layer: fast and strict encodings identical (every plane, scale, bias, ratio
    index and MSE); the contract on 32 sampled groups against the oracle."""
    M, N = 1024, 4096
    W = synthetic.gaussian_weight(M, N, seed=77, sigma=0.02)
    Wd = torch.from_numpy(W).to(DEV)
    wf, mf = sb.encode_weights(Wd, K=4, strict=False, return_mse=True)
    ws, ms = sb.encode_weights(Wd, K=4, strict=True, return_mse=True)
    torch.cuda.synchronize()
    assert torch.equal(wf.data, ws.data) and torch.equal(mf, ms)
    pc, s16, b16, ri = sb.unpack_canonical(wf)
    R = oracle.ratio_set(16)
    cfg = oracle.OracleConfig()
    for q in np.random.default_rng(3).choice(M * (N // 128), 32, replace=False):
        r, g = divmod(int(q), N // 128)
        X = W[r, 128 * g:128 * (g + 1)].astype(np.float64)
        best = oracle.encode_group(X, cfg)["mse"]
        m = oracle.entry_mse(X, 4, float(R[ri[r, g]]), _fp16(s16[r, g]), _fp16(b16[r, g]))
        assert m <= best * (1 + 1e-6) and mf[r, g].item() == m


def test_encode_fast_rejected_where_not_built():
    W = torch.zeros(16, 128, device=DEV)
    cfg_kw = dict(K=4, n_ratio=16, n_scale=64, n_bias=16)
    with pytest.raises(sb.SbvrError) as e:
        sb.encode_weights_cached(W, strict=False, **cfg_kw)
    assert e.value.status == sb.ERR_UNSUPPORTED
