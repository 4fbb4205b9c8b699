"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bar: bit-exact for planes, meta, activation planes/scales and popcount partials;
float y within max normwise relative error 1e-3 and per-element floored relative error 1e-3
against the fp64 oracle.  Inputs are seeded and synthetic (synthetic/), shared by both sides.
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


def rel_errors(y, ref):
    y = np.asarray(y, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(y - ref)
    scale = np.abs(ref).max() if ref.size else 1.0
    scale = scale if scale > 0 else 1.0
    normwise = err.max() / scale if err.size else 0.0
    floored = (err / np.maximum(np.abs(ref), 1e-2 * scale)).max() if err.size else 0.0
    return normwise, floored


def assert_close(y, ref):
    nw, fl = rel_errors(y, ref)
    assert nw <= TOL and fl <= TOL, (nw, fl)


def _oracle_encoded(pc, s16, b16, ri, K, n_ratio):
    M, NG = s16.shape
    return oracle.Encoded(M, NG * 128, oracle.OracleConfig(K=K, n_ratio=n_ratio), pc, s16, b16, ri, np.zeros((M, NG)))


# ------------------------------------------------------------------ a4: activation conversion (bit-exact)
@pytest.mark.parametrize("T,N,l", [(1, 128, 8), (1, 4096, 8), (3, 1024, 8), (2, 512, 4), (1, 14336, 8), (16, 4096, 8)])
def test_encode_vector_bitexact(T, N, l):
    x = synthetic.activation(N, seed=N + T + l, T=T, outliers=3)
    if N >= 256:
        x[0, :128] = 0                                   # all-zero group
        x[0, 128] = 127.0                                # absmax 127 -> s_x = 1: exact RNE ties below
        x[0, 129:133] = [2.5, 3.5, -2.5, 0.5]
    act = sb.encode_vector(torch.from_numpy(x).to(DEV), l=l)
    torch.cuda.synchronize()
    planes = act.data.cpu().numpy().view(np.uint32).reshape(T, N // 128, l, 4)
    scales = act.scales.cpu().numpy().reshape(T, N // 128)
    for t in range(T):
        z, op, osc = oracle.encode_vector(x[t], 128, l)
        assert np.array_equal(planes[t], op)
        assert np.array_equal(scales[t].view(np.uint32), osc.view(np.uint32))


# ------------------------------------------------------------------ a1-a3: encoder (bit-exact, strict fp64)
@pytest.mark.parametrize("K,dtype", [(4, torch.float32), (3, torch.float32), (2, torch.bfloat16), (4, torch.float16)])
def test_encode_weights_bitexact_small(K, dtype):
    M, N = 32, 256                                       # 64 groups, 2 row tiles, 2 groups per row
    W = synthetic.with_degenerate_groups(synthetic.gaussian_weight(M, N, seed=K, sigma=0.02), seed=K)
    Wt = torch.from_numpy(W).to(dtype)
    cfg = oracle.OracleConfig(K=K, n_ratio=16, n_scale=64 if K == 4 else 16, n_bias=16)
    w, mse = sb.encode_weights(Wt.to(DEV), K=K, n_ratio=cfg.n_ratio, n_scale=cfg.n_scale, n_bias=cfg.n_bias,
                               return_mse=True)
    torch.cuda.synchronize()
    ref = oracle.encode_matrix(Wt.float().numpy(), cfg)
    pc, s16, b16, ri = sb.unpack_canonical(w)
    assert np.array_equal(pc, ref.planes)
    assert np.array_equal(s16, ref.s16) and np.array_equal(b16, ref.b16) and np.array_equal(ri, ref.r_idx)
    assert np.array_equal(mse.cpu().numpy(), ref.mse)
    # ratio table = r^t of the oracle's R in fp32
    R = oracle.ratio_set(cfg.n_ratio)
    assert np.allclose(w.ratio_pow.cpu().numpy(), np.power(R[:, None], np.arange(K)[None, :]), rtol=1e-7)


def test_encode_weights_sampled_groups_full_size():
    """Llama-3-8B q_proj shape: GPU encodes all 131072 groups; the oracle re-encodes 24 sampled ones."""
    M, N = 4096, 4096
    W = synthetic.gaussian_weight(M, N, seed=100, sigma=0.02)
    w = sb.encode_weights(torch.from_numpy(W).to(DEV), K=4)
    torch.cuda.synchronize()
    pc, s16, b16, ri = sb.unpack_canonical(w)
    rng = np.random.default_rng(0)
    cfg = oracle.OracleConfig()
    for q in rng.choice(M * (N // 128), 24, replace=False):
        r, g = divmod(int(q), N // 128)
        ref = oracle.encode_group(W[r, 128 * g:128 * (g + 1)].astype(np.float64), cfg)
        assert np.array_equal(pc[r, g], ref["planes"]) and s16[r, g] == ref["s16"] and b16[r, g] == ref["b16"]
        assert ri[r, g] == ref["r_idx"]


def test_encode_weights_deterministic():
    W = torch.from_numpy(synthetic.gaussian_weight(64, 512, seed=7)).to(DEV)
    a = sb.encode_weights(W, K=4, n_scale=16)
    b = sb.encode_weights(W, K=4, n_scale=16)
    torch.cuda.synchronize()
    assert torch.equal(a.data, b.data) and torch.equal(a.ratio_pow, b.ratio_pow)


# ------------------------------------------------------------------ a5/a7: SBVR-x GEMV (partials bit-exact, y to 1e-3)
SHAPES = [(16, 128), (64, 256), (80, 384), (208, 1024), (1024, 512), (336, 640), (272, 256)]


@pytest.mark.parametrize("M,N", SHAPES)
@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("algo", [sb.ALGO_PIPE, sb.ALGO_MMA, sb.ALGO_TC, sb.ALGO_POPC])
def test_gemv_sbvr_x(M, N, K, algo):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M * 7 + N + K)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=N + 1)
    act = sb.encode_vector(torch.from_numpy(x).to(DEV))
    y = sb.gemv_ex(w, act, algo=algo)
    P = sb.debug_partials(w, act, algo=algo)
    torch.cuda.synchronize()
    z, xp, sc = oracle.encode_vector(x[0], 128, 8)
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    ref = oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc))
    assert_close(y.cpu().numpy()[0], ref)
    Pref, _ = oracle.partials_rows(enc, z, xp)
    assert np.array_equal(P.cpu().numpy(), Pref)


@pytest.mark.parametrize("l", [8, 6, 5, 4, 2])
@pytest.mark.parametrize("algo", [sb.ALGO_PIPE, sb.ALGO_MMA, sb.ALGO_TC])
def test_gemv_sbvr_x_activation_bits(l, algo):
    M, N, K = 48, 256, 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=l)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=l)
    act = sb.encode_vector(torch.from_numpy(x).to(DEV), l=l)
    y = sb.gemv_ex(w, act, algo=algo)
    P = sb.debug_partials(w, act, algo=algo)
    torch.cuda.synchronize()
    z, xp, sc = oracle.encode_vector(x[0], 128, l)
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    assert_close(y.cpu().numpy(), oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
    Pref, _ = oracle.partials_rows(enc, z, xp, l=l)
    assert np.array_equal(P.cpu().numpy(), Pref)


def test_gemv_on_gpu_encoded_weights_matches_oracle_end_to_end():
    """Oracle encodes W and computes y; the GPU encodes the same W and computes y."""
    M, N, K = 48, 384, 4
    W = synthetic.gaussian_weight(M, N, seed=31, sigma=0.02)
    x = synthetic.activation(N, seed=32)
    cfg = oracle.OracleConfig(n_scale=16)
    enc = oracle.encode_matrix(W, cfg)
    z, xp, sc = oracle.encode_vector(x[0], 128, 8)
    w = sb.encode_weights(torch.from_numpy(W).to(DEV), K=K, n_scale=16)
    act = sb.encode_vector(torch.from_numpy(x).to(DEV))
    y = sb.gemv(w, act)
    yf = sb.gemv(w, sb.fp16_activation(torch.from_numpy(x[0]).to(DEV)))
    torch.cuda.synchronize()
    assert_close(y.cpu().numpy(), oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
    assert_close(yf.cpu().numpy(), oracle.gemv_rows(enc, oracle.x_dec_fp16(x[0])))


# ------------------------------------------------------------------ a6: fp16-x GEMV
@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (80, 384, 3), (256, 1024, 2), (336, 640, 4), (1024, 512, 4)])
@pytest.mark.parametrize("algo", [sb.ALGO_AUTO, sb.ALGO_POPC])
def test_gemv_fp16_x(M, N, K, algo):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M + N)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=3)
    y = sb.gemv_ex(w, sb.fp16_activation(torch.from_numpy(x[0]).to(DEV)), algo=algo)[0]
    torch.cuda.synchronize()
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    assert_close(y.cpu().numpy(), oracle.gemv_rows(enc, oracle.x_dec_fp16(x[0])))


# ------------------------------------------------------------------ a8: batched
@pytest.mark.parametrize("T", [1, 2, 3, 4, 5, 8, 16])
@pytest.mark.parametrize("algo", [sb.ALGO_AUTO, sb.ALGO_MMA, sb.ALGO_TC])
def test_gemv_batched(T, algo):
    M, N, K = 208, 512, 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=T)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=T + 50, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV))
    Y = sb.gemv_ex(w, act, algo=algo)
    Yf = sb.gemv_ex(w, sb.fp16_activation(torch.from_numpy(X).to(DEV)))
    torch.cuda.synchronize()
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    for t in range(T):
        z, xp, sc = oracle.encode_vector(X[t], 128, 8)
        assert_close(Y.cpu().numpy()[t], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
        assert_close(Yf.cpu().numpy()[t], oracle.gemv_rows(enc, oracle.x_dec_fp16(X[t])))


# ------------------------------------------------------------------ full-size shapes, sampled rows, bench launch config
@pytest.mark.parametrize("name,M,N", synthetic.LLAMA3_8B_LAYER + [("70b_down", 8192, 28672),
                                                                   ("gate_up_fused", 28672, 4096),
                                                                   ("tall_narrow", 16384, 256)])
@pytest.mark.parametrize("algo", [sb.ALGO_PIPE, sb.ALGO_MMA, sb.ALGO_TC])
def test_gemv_full_size_sampled_rows(name, M, N, algo):
    K = 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M ^ N)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=11)
    act = sb.encode_vector(torch.from_numpy(x).to(DEV))
    ws = sb.Workspace.for_weights(w, 1)
    y = sb.gemv_ex(w, act, ws=ws, algo=algo)[0]
    y2 = sb.gemv_ex(w, act, ws=ws, algo=algo)[0]   # workspace reuse: counters must have been reset
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([np.random.default_rng(1).choice(M, 200, replace=False), [0, M - 1, 63, 64]]))
    z, xp, sc = oracle.encode_vector(x[0], 128, 8)
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    ref = oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows)
    yy = y.cpu().numpy()
    assert_close(yy[rows], ref)
    assert torch.equal(y, y2)                # deterministic
    P = sb.debug_partials(w, act, algo=algo)
    Pref, _ = oracle.partials_rows(enc, z, xp, rows=rows[:16])
    assert np.array_equal(P.cpu().numpy()[rows[:16]], Pref)
    if algo == sb.ALGO_MMA:                       # fp16-x path on the same weights, same launch config
        yf = sb.gemv_ex(w, sb.fp16_activation(torch.from_numpy(x[0]).to(DEV)), ws=ws)[0]
        torch.cuda.synchronize()
        assert_close(yf.cpu().numpy()[rows], oracle.gemv_rows(enc, oracle.x_dec_fp16(x[0]), rows))


def test_pipe_ticket_counter_rearmed_across_launches():
    """The persistent kernel's dynamic work counter and partial slots must be back at rest after
    every launch: many back-to-back launches on one workspace (different shapes), every result
    checked against the oracle and against a re-run."""
    ws = sb.Workspace(64 << 20)
    for i, (M, N) in enumerate([(4096, 4096), (1024, 4096), (16, 128), (6144, 4096), (4096, 14336), (4096, 4096)]):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=100 + i)
        w = sb.pack_canonical(pc, s16, b16, ri, 16)
        x = synthetic.activation(N, seed=200 + i)
        act = sb.encode_vector(torch.from_numpy(x).to(DEV))
        ys = [sb.gemv_ex(w, act, ws=ws, algo=sb.ALGO_PIPE)[0] for _ in range(3)]
        torch.cuda.synchronize()
        assert all(torch.equal(ys[0], y) for y in ys[1:])
        rows = np.unique(np.concatenate([np.random.default_rng(i).choice(M, min(M, 64), replace=False), [0, M - 1]]))
        z, xp, sc = oracle.encode_vector(x[0], 128, 8)
        enc = _oracle_encoded(pc, s16, b16, ri, 4, 16)
        assert_close(ys[0].cpu().numpy()[rows], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc), rows))
    assert torch.all(ws.buf.view(torch.int32) == -1)   # every slot and the counter re-armed


# ------------------------------------------------------------------ error behaviour
def test_abi_errors():
    pc, s16, b16, ri = synthetic.random_encoded(32, 256, 4, 16, seed=0)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    act = sb.encode_vector(torch.zeros(384, dtype=torch.float16, device=DEV))
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv(w, act)
    assert e.value.status == sb.ERR_SHAPE
    # a matrix split over many CTAs needs cross-CTA slots: a 256-byte workspace is too small
    pcb, s16b, b16b, rib = synthetic.random_encoded(1024, 4096, 4, 16, seed=1)
    wb = sb.pack_canonical(pcb, s16b, b16b, rib, 16)
    assert sb.Workspace.for_weights(wb, 1).nbytes > 256
    actb = sb.encode_vector(torch.zeros(4096, dtype=torch.float16, device=DEV))
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv(wb, actb, ws=sb.Workspace(256))
    assert e.value.status == sb.ERR_WORKSPACE
    act = sb.encode_vector(torch.zeros(256, dtype=torch.float16, device=DEV))
    y = sb.gemv(w, act)
    torch.cuda.synchronize()
    assert not y.any()                       # zero activation -> zero output


# ------------------------------------------------------------------ f4: randomized Hadamard rotation
@pytest.mark.parametrize("rows,N,b", [(1, 32, 32), (3, 256, 64), (17, 1024, 128), (5, 4096, 1024), (33, 14336, 512),
                                      (2, 768, 256)])
@pytest.mark.parametrize("dt", [torch.float32, torch.float16])
def test_hadamard_rows(rows, N, b, dt):
    """Tolerance: fp32 butterflies add at most log2(b) roundings per output (<= 10 x 2^-24 relative to
    the block norm), so 1e-5 normwise; fp16 output rounding adds 2^-11 relative -> 1e-3."""
    W = synthetic.student_t_weight(rows, N, seed=rows + N).astype(np.float32)
    if dt == torch.float16:
        W = W.astype(np.float16).astype(np.float32)
    s = synthetic.hadamard_signs(N, seed=b)
    X = torch.from_numpy(W).to(DEV).to(dt)
    sg = torch.from_numpy(s).to(DEV)
    Y = sb.hadamard_rows(X, sg, block=b)
    Xi = X.clone()
    sb.hadamard_rows(Xi, sg, block=b, out=Xi)            # in place
    torch.cuda.synchronize()
    ref = oracle.hadamard_rows(W.astype(np.float64), s, b)
    err = np.abs(Y.double().cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= (1e-5 if dt == torch.float32 else 1e-3), err
    assert torch.equal(Y, Xi)


def test_hadamard_errors():
    X = torch.zeros(2, 96, device=DEV)
    sg = torch.ones(96, dtype=torch.int8, device=DEV)
    with pytest.raises(sb.SbvrError) as e:
        sb.hadamard_rows(X, sg, block=96)
    assert e.value.status == sb.ERR_UNSUPPORTED
    with pytest.raises(sb.SbvrError) as e:
        sb.hadamard_rows(X, sg, block=64)
    assert e.value.status == sb.ERR_SHAPE


def test_hadamard_then_encode_lowers_heavy_tail_mse():
    """f4's effect: encoding Student-t(3) weights after the 128-block rotation gives a lower mean
    group MSE (the rotation is orthogonal, so the rotated-domain MSE is the original-domain MSE)."""
    W = torch.from_numpy(synthetic.student_t_weight(64, 1024, seed=77)).to(DEV)
    sg = torch.from_numpy(synthetic.hadamard_signs(1024, seed=78)).to(DEV)
    _, mse0 = sb.encode_weights(W, K=4, n_scale=16, return_mse=True)
    _, mse1 = sb.encode_weights(sb.hadamard_rows(W, sg, block=128), K=4, n_scale=16, return_mse=True)
    torch.cuda.synchronize()
    assert mse1.mean().item() < mse0.mean().item()


@pytest.mark.parametrize("T,l", [(3, 8), (8, 8), (8, 5), (11, 4), (16, 8)])
def test_gemv_batched_z_columns(T, l):
    """Batches on the z-column formulation (MMA path, T >= 3: B = z (s8) of 8 tokens, A = plane bits 0/1,
    T_t read from the accumulator), incl. l < 8 (sign-extended planes) and a ragged last pass."""
    M, N, K = 336, 640, 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=T * 10 + l)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = synthetic.activation(N, seed=T + l, T=T)
    act = sb.encode_vector(torch.from_numpy(X).to(DEV), l=l)
    Y = sb.gemv_ex(w, act, algo=sb.ALGO_MMA)
    torch.cuda.synchronize()
    enc = _oracle_encoded(pc, s16, b16, ri, K, 16)
    for t in range(T):
        z, xp, sc = oracle.encode_vector(X[t], 128, l)
        assert_close(Y.cpu().numpy()[t], oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))


@pytest.mark.parametrize("T", [3, 5, 6, 7, 9])
@pytest.mark.parametrize("kind", ["sbvr", "fp16"])
@pytest.mark.parametrize("algo", [sb.ALGO_AUTO, sb.ALGO_MMA, sb.ALGO_TC])
def test_batched_writes_stay_inside_y(T, kind, algo):
    """Passes that keep 8 (or 4) token columns must not write rows of Y beyond T."""
    if kind == "fp16" and algo == sb.ALGO_TC:
        pytest.skip("fp16-x runs on MMA/POPC")
    M, N, K = 208, 512, 4
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=T)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    X = torch.from_numpy(synthetic.activation(N, seed=T, T=T)).to(DEV)
    act = sb.encode_vector(X) if kind == "sbvr" else sb.fp16_activation(X)
    big = torch.full((T + 8, M), 12345.0, device=DEV)
    sb.gemv_ex(w, act, y=big[:T], algo=algo)
    torch.cuda.synchronize()
    assert torch.all(big[T:] == 12345.0)
    assert torch.isfinite(big[:T]).all()


# ------------------------------------------------------------------ f2: encode-time coefficient cache
@pytest.mark.parametrize("K,cache_size,M,N", [(4, 8, 16, 1024), (3, 4, 16, 512), (2, 16, 32, 1024), (4, 0, 16, 512)])
def test_encode_weights_cached_bitexact(K, cache_size, M, N):
    """Planes, fp16 meta, ratio index, fp64 group MSE and the hit flags of the cached encoder equal the
    oracle's (reading A22), incl. degenerate groups; cache_size 0 equals the uncached encoder."""
    W = synthetic.with_degenerate_groups(synthetic.gaussian_weight(M, N, seed=K * 100 + M, sigma=0.02), seed=K)
    cfg = oracle.OracleConfig(K=K, n_scale=16)
    enc, hit = oracle.encode_matrix_cached(W, cfg, cache_size=cache_size, alpha=0.1)
    w, mse, h = sb.encode_weights_cached(torch.from_numpy(W).to(DEV), K=K, cache_size=cache_size, ema_alpha=0.1,
                                         n_scale=16)
    torch.cuda.synchronize()
    pc, s16, b16, ri = sb.unpack_canonical(w)
    assert np.array_equal(h.cpu().numpy(), hit)
    assert np.array_equal(pc, enc.planes) and np.array_equal(s16, enc.s16) and np.array_equal(b16, enc.b16)
    assert np.array_equal(ri, enc.r_idx) and np.array_equal(mse.cpu().numpy(), enc.mse)
    if cache_size == 0:
        w0 = sb.encode_weights(torch.from_numpy(W).to(DEV), K=K, n_scale=16)
        torch.cuda.synchronize()
        assert torch.equal(w0.data, w.data)
