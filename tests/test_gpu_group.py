"""GPU parity of sbvr_gemv_group (include/sbvr.h): independent batch-1 SBVR-x GEMVs in one persistent
launch.  Every y against the fp64 oracle (SURVEY §8c.5 bar, normwise and floored relative error <= 1e-3): small
problems element by element (several matrices of different N, ragged unit counts, problems smaller than one CTA's
share, bands split across CTAs and across problem boundaries), the bench step's layer set at full size on sampled
rows, CUDA-graph replay, determinism, workspace at rest (with a canary after it), K = 2/3/4, and the ABI's
rejections.  Also: the grouped y agrees with per-problem sbvr_gemv to fp32 reduction-order rounding.
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


def _make(M, N, K, seed, l=8):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=seed)
    w = sb.pack_canonical(pc, s16, b16, ri, 16)
    x = synthetic.activation(N, seed=seed + 1)[0]
    act = sb.encode_vector(torch.from_numpy(x).to(DEV), l=l)
    enc = oracle.Encoded(M, N, oracle.OracleConfig(K=K, n_ratio=16), pc, s16, b16, ri, None)
    z, _, sc = oracle.encode_vector(x, 128, l)
    return w, act, enc, oracle.x_dec_sbvr(z, sc)


class _CanaryWs:
    CANARY = 4096

    def __init__(self, problems):
        n = sb.group_workspace(problems).nbytes
        self.full = torch.full((n + self.CANARY,), 0x5A, dtype=torch.uint8, device=DEV)
        self.buf = self.full[:n]
        self.nbytes = n
        self.buf.fill_(0xFF)

    def canary_ok(self):
        return bool(torch.all(self.full[self.nbytes:] == 0x5A))

    def ok(self):
        return self.canary_ok() and bool(torch.all(self.buf == 0xFF))


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("shapes", [
    [(128, 128)],                                   # one unit pair: a single tiny problem
    [(256, 512), (128, 1280), (384, 384)],          # different N, few units: bands shared across CTAs
    [(640, 1024), (128, 128), (1280, 640), (256, 2048), (128, 256)],   # ragged mix, a 2-unit problem inside
])
def test_group_small_elementwise(K, shapes):
    probs, refs = [], []
    for i, (M, N) in enumerate(shapes):
        w, act, enc, xd = _make(M, N, K, seed=100 * K + 10 * i + len(shapes))
        probs.append((w, act, torch.full((M,), float("nan"), device=DEV)))
        refs.append(oracle.gemv_rows(enc, xd))
    ws = _CanaryWs(probs)
    ys = sb.gemv_group(probs, ws=ws)
    ys2 = [y.clone() for y in ys]
    sb.gemv_group(probs, ws=ws)                    # workspace reuse, determinism
    torch.cuda.synchronize()
    assert ws.ok()
    for y, y2, ref in zip(ys, ys2, refs):
        assert torch.equal(y, y2)
        _close(y.cpu().numpy(), ref)


def test_group_matches_single_launch():
    """Same arithmetic as sbvr_gemv's MMA kernel: the grouped y differs from the single-launch y only by the fp32
    order in which split-K band partials are added (relative 1e-6)."""
    probs = []
    for i, (M, N) in enumerate([(1024, 4096), (4096, 4096), (2048, 14336)]):
        w, act, _, _ = _make(M, N, 4, seed=300 + i)
        probs.append((w, act, None))
    ys = sb.gemv_group(probs)
    for (w, act, _), y in zip(probs, ys):
        y1 = sb.gemv(w, act)
        torch.cuda.synchronize()
        d = (y - y1).abs().max().item() / max(y1.abs().max().item(), 1e-30)
        assert d < 1e-5, d


FUSED = [(6144, 4096, 0), (4096, 4096, 1), (28672, 4096, 2), (4096, 14336, 3)]
INPUT_N = [4096, 4096, 4096, 14336]


def _rows(M, seed, n=64):
    r = np.random.default_rng(seed).choice(M, min(M, n), replace=False)
    edges = [0, M - 1] + [b for b in (63, 64, 127, 128, M // 2) if b < M]
    return np.unique(np.concatenate([r, edges]))


def test_group_bench_step_graph_parity():
    """The bench's grouped step: one sbvr_encode_vector over the 4 concatenated layer inputs + one sbvr_gemv_group
    over the layer set (fused qkv, o, fused gate_up, down), captured as CUDA graphs over a 2-layer ring, each
    replayed 3 times; every y on sampled rows against the oracle, replays bit-identical."""
    ring = 2
    layers = []
    for r in range(ring):
        mats = []
        for j, (M, N, xin) in enumerate(FUSED):
            pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=700 + 10 * r + j)
            w = sb.pack_canonical(pc, s16, b16, ri, 16)
            enc = oracle.Encoded(M, N, oracle.OracleConfig(K=4, n_ratio=16), pc, s16, b16, ri, None)
            mats.append((w, torch.full((M,), float("nan"), device=DEV), xin, enc))
        layers.append(mats)
    xs = [synthetic.activation(n, seed=710 + i)[0] for i, n in enumerate(INPUT_N)]
    xcat = torch.from_numpy(np.concatenate(xs)).to(DEV)
    act_all = sb.encode_vector(xcat)
    acts, g0 = [], 0
    for n in INPUT_N:
        ng = n // 128
        acts.append(sb.SbvrActivation(sb.ACT_SBVR, n, 1, 8, act_all.data[g0 * 32:(g0 + ng) * 32], act_all.scales[g0:g0 + ng]))
        g0 += ng
    probs = [[(w, acts[xin], y) for (w, y, xin, _) in layers[r]] for r in range(ring)]
    wss = [_CanaryWs(probs[r]) for r in range(ring)]
    stream = torch.cuda.Stream()
    graphs = []
    with torch.cuda.stream(stream):
        def step(r):
            sb.encode_vector(xcat, out=act_all)
            sb.gemv_group(probs[r], ws=wss[r])
        step(0)
        torch.cuda.synchronize()
        for r in range(ring):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step(r)
            graphs.append(g)
        for (_, y, _, _) in layers[0] + layers[1]:
            y.fill_(float("nan"))
        outs = []
        for it in range(3 * ring):
            graphs[it % ring].replay()
            outs.append([y.clone() for (_, y, _, _) in layers[it % ring]])
    torch.cuda.synchronize()
    assert all(w.ok() for w in wss)
    xdec = []
    for x in xs:
        z, xp, sc = oracle.encode_vector(x, 128, 8)
        xdec.append(oracle.x_dec_sbvr(z, sc))
    for it, ys in enumerate(outs):
        r = it % ring
        for j, ((w, _, xin, enc), y) in enumerate(zip(layers[r], ys)):
            rows = _rows(w.M, it + 10 * j)
            _close(y.cpu().numpy()[rows], oracle.gemv_rows(enc, xdec[xin], rows))
            if it >= ring:
                assert torch.equal(y, outs[it - ring][j])


def test_group_rejections():
    w, act, _, _ = _make(128, 256, 4, seed=5)
    w1, act1, _, _ = _make(128, 256, 1, seed=6)
    y = torch.empty(128, device=DEV)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_group([(w, sb.fp16_activation(torch.zeros(256, dtype=torch.float16, device=DEV)), y)])
    assert e.value.status == sb.ERR_UNSUPPORTED
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_group([(w1, act1, y)])                   # K = 1
    assert e.value.status == sb.ERR_UNSUPPORTED
    w3, act3, _, _ = _make(128, 256, 3, seed=7)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_group([(w, act, y), (w3, act3, torch.empty(128, device=DEV))])   # K differs
    assert e.value.status == sb.ERR_UNSUPPORTED
    w64, act64, _, _ = _make(64, 256, 4, seed=8)
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_group([(w64, act64, torch.empty(64, device=DEV))])               # M % 128 != 0
    assert e.value.status == sb.ERR_SHAPE
    with pytest.raises(sb.SbvrError) as e:
        sb.gemv_group([(w, act, y)] * 9)
    assert e.value.status == sb.ERR_INVALID_ARG


@pytest.mark.parametrize("l", [8, 4])
def test_group_in_kernel_conversion_bit_identical(l):
    """SBVR_ACT_FP16_Q problems: the kernel converts every problem's fp16 x itself (Eq. 12, distributed over the
    grid, then a grid-wide arrival count) -- y bit-identical to sbvr_encode_vector + the grouped GEMV on SBVR-x,
    every y within the oracle bar, the workspace (conversion counters included) back at rest, several launches."""
    shapes = [(1024, 4096), (4096, 4096), (2048, 14336), (256, 384)]
    probs_q, probs_s, refs = [], [], []
    for i, (M, N) in enumerate(shapes):
        pc, s16, b16, ri = synthetic.random_encoded(M, N, 4, 16, seed=500 + i)
        w = sb.pack_canonical(pc, s16, b16, ri, 16)
        x = synthetic.activation(N, seed=510 + i, outliers=8 if i == 1 else 0)[0]
        xd = torch.from_numpy(x).to(DEV)
        probs_q.append((w, sb.fp16q_activation(xd, l=l), torch.full((M,), float("nan"), device=DEV)))
        probs_s.append((w, sb.encode_vector(xd, l=l), torch.full((M,), float("nan"), device=DEV)))
        enc = oracle.Encoded(M, N, oracle.OracleConfig(K=4, n_ratio=16), pc, s16, b16, ri, None)
        z, _, sc = oracle.encode_vector(x, 128, l)
        refs.append(oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc)))
    ws = _CanaryWs(probs_q)
    ys_s = sb.gemv_group(probs_s)
    for it in range(3):
        ys_q = sb.gemv_group(probs_q, ws=ws)
        torch.cuda.synchronize()
        assert ws.canary_ok()          # (the conversion scratch holds the converted x; counters re-armed: next launch)
        for yq, ys in zip(ys_q, ys_s):
            assert torch.equal(yq, ys)
    for y, ref in zip(ys_q, refs):
        _close(y.cpu().numpy(), ref)
