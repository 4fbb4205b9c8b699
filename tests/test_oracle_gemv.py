"""Pins for the activation (O-X), GEMV (O-Y) and popcount-partials (O-P) oracle steps.

Pins: the worked examples in tests/golden/ (SPEC S:315), RNE ties, the round-trip
bound |x - z s| <= s/2, the two's-complement identity sum_j alpha_j d_j = z, popcount of
ANDed words (an independent route to P), exact 0-ulp agreement of decode-then-dot
(O-Y) with the AND/popcount form (O-Y') on dyadic inputs, one-hot rows and bilinearity.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
ALPHA8 = np.array([1, 2, 4, 8, 16, 32, 64, -128], np.int64)


# ------------------------------------------------------------------ O-X activation conversion (Eq. 12)
def test_activation_spec_example():
    g = SPEC["activation"]
    x = np.zeros(128, np.float16)
    x[0] = g["absmax"]
    x[5] = g["element"]
    z, planes, scales = oracle.encode_vector(x, 128, g["l"])
    assert z[5] == g["z"]
    bits = [(int(planes[0, j, 0]) >> 5) & 1 for j in range(8)]
    assert bits == g["bits_lsb_first"]
    assert z[0] == 127


def test_activation_rne_ties():
    x = np.zeros(128, np.float16)
    x[0] = 127.0          # absmax 127 -> s_x = 1 exactly
    x[1], x[2], x[3], x[4] = 2.5, 3.5, -2.5, 0.5
    z, _, s = oracle.encode_vector(x, 128, 8)
    assert s[0] == 1.0
    assert (z[1], z[2], z[3], z[4]) == (2, 4, -2, 0)   # round half to even (reading A12)


def test_activation_round_trip_and_twos_complement():
    rng = np.random.default_rng(20)
    for l in (8, 6, 4):
        zmax = 2 ** (l - 1) - 1
        alpha = np.array([2 ** j for j in range(l - 1)] + [-(2 ** (l - 1))], np.int64)
        for _ in range(20):
            x = (rng.standard_normal(512) * rng.uniform(0.01, 10)).astype(np.float16)
            z, planes, s = oracle.encode_vector(x, 128, l)
            xs = x.astype(np.float64)
            for g in range(4):
                seg = slice(128 * g, 128 * (g + 1))
                assert s[g] == np.float32(np.float32(np.abs(x[seg]).astype(np.float32).max()) / np.float32(zmax))
                err = np.abs(xs[seg] - z[seg] * np.float64(s[g]))
                assert np.all(err <= s[g] / 2 * (1 + 1e-6))
                assert np.abs(z[seg]).max() == zmax and np.abs(z[seg]).max() <= zmax
                for e in range(128):
                    d = [(int(planes[g, j, e // 32]) >> (e % 32)) & 1 for j in range(l)]
                    assert int(np.dot(alpha, d)) == z[128 * g + e]


def test_activation_zero_group():
    x = np.zeros(256, np.float16)
    x[200] = 1.0
    z, planes, s = oracle.encode_vector(x, 128, 8)
    assert s[0] == 0.0 and not z[:128].any() and not planes[0].any()
    assert s[1] > 0


# ------------------------------------------------------------------ helpers to build encoded matrices by hand
def _enc(M, N, K, n_ratio, planes, s, b, ridx):
    cfg = oracle.OracleConfig(K=K, n_ratio=n_ratio)
    NG = N // 128
    s16 = np.array([[oracle.fp16_bits(v) for v in row] for row in np.broadcast_to(s, (M, NG))], np.uint16)
    b16 = np.array([[oracle.fp16_bits(v) for v in row] for row in np.broadcast_to(b, (M, NG))], np.uint16)
    return oracle.Encoded(M, N, cfg, np.ascontiguousarray(planes, np.uint32), s16, b16,
                          np.ascontiguousarray(np.broadcast_to(ridx, (M, NG)), np.uint8), np.zeros((M, NG)))


def test_gemv_worked_example_spec_s364():
    g = SPEC["inner_product"]
    R = oracle.ratio_set(16)
    ridx = int(np.where(R == 0.5)[0][0])         # c = (1, 0.5, 0.25) = s r^t + b with s=1, r=0.5, b=0
    planes = np.zeros((1, 1, 3, 4), np.uint32)
    for t, bit in enumerate(g["w_bits"]):
        planes[0, 0, t, 0] = bit
    enc = _enc(1, 128, 3, 16, planes, 1.0, 0.0, ridx)
    x = np.zeros(128)
    x[0] = g["x_value"]
    assert oracle.gemv_rows(enc, x)[0] == g["result"]


def test_gemv_one_hot_rows_and_zero():
    M, N, K = 8, 256, 4
    planes = np.zeros((M, 2, K, 4), np.uint32)
    cols = [3, 77, 128, 255, 0, 31, 32, 200]
    for r, c in enumerate(cols):
        planes[r, c // 128, 0, (c % 128) // 32] = 1 << (c % 32)   # only plane 0 set -> w = c_0 = s + b = 1
    enc = _enc(M, N, K, 4, planes, 1.0, 0.0, 1)
    x = np.random.default_rng(21).standard_normal(N)
    assert np.array_equal(oracle.gemv_rows(enc, x), x[cols])
    assert not oracle.gemv_rows(enc, np.zeros(N)).any()
    assert np.array_equal(oracle.gemv_rows(enc, 4 * x), 4 * x[cols])      # bilinearity, exact for 2^k


def _random_enc(rng, M, N, K, n_ratio, dyadic):
    NG = N // 128
    planes = rng.integers(0, 2 ** 32, (M, NG, K, 4), dtype=np.uint64).astype(np.uint32)
    if dyadic:
        s = rng.integers(1, 64, (M, NG)) / 64.0
        b = rng.integers(-16, 16, (M, NG)) / 256.0
    else:
        s = rng.uniform(0.01, 0.1, (M, NG))
        b = rng.uniform(-0.01, 0.01, (M, NG))
    ridx = rng.integers(0, n_ratio, (M, NG))
    return _enc(M, N, K, n_ratio, planes, s, b, ridx)


def _y_popcount_form(enc, P, scales):
    """O-Y': y = sum_g s_x sum_t c_t sum_j alpha_j P_tj."""
    R = oracle.ratio_set(enc.cfg.n_ratio)
    M, NG, K = P.shape[0], P.shape[1], P.shape[2]
    y = np.zeros(M)
    for r in range(M):
        acc = 0.0
        for g in range(NG):
            c = oracle.coefficients(R[enc.r_idx[r, g]], oracle.fp16_to_double(enc.s16[r, g]),
                                    oracle.fp16_to_double(enc.b16[r, g]), K)
            for t in range(K):
                T = int(np.dot(ALPHA8, P[r, g, t].astype(np.int64)))
                acc += float(scales[g]) * c[t] * T
        y[r] = acc
    return y


def test_gemv_equals_popcount_form_exactly_on_dyadic_inputs():
    """North star: 'the identity that the AND/popcount inner product equals the decoded fp64 dot product'."""
    rng = np.random.default_rng(22)
    for K in (2, 3, 4):
        enc = _random_enc(rng, 6, 512, K, 4, dyadic=True)      # R = {-1, -0.5, 0.5, 1}
        x = np.zeros(512, np.float16)
        for g in range(4):                                      # absmax 127 * 2^-k -> s_x = 2^-k exactly
            x[128 * g:128 * (g + 1)] = (rng.integers(-127, 128, 128) * 2.0 ** -(g + 2)).astype(np.float16)
            x[128 * g] = 127 * 2.0 ** -(g + 2)
        z, xp, sc = oracle.encode_vector(x, 128, 8)
        assert all(sc[g] == 2.0 ** -(g + 2) for g in range(4))
        P, T = oracle.partials_rows(enc, z, xp)
        y = oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc))
        assert np.array_equal(y, _y_popcount_form(enc, P, sc))


def test_gemv_equals_popcount_form_general():
    rng = np.random.default_rng(23)
    enc = _random_enc(rng, 5, 384, 4, 16, dyadic=False)
    x = rng.standard_normal(384).astype(np.float16)
    z, xp, sc = oracle.encode_vector(x, 128, 8)
    P, T = oracle.partials_rows(enc, z, xp)
    y = oracle.gemv_rows(enc, oracle.x_dec_sbvr(z, sc))
    assert np.allclose(y, _y_popcount_form(enc, P, sc), rtol=1e-12, atol=1e-14)
    W = oracle.decode_matrix(enc)
    assert np.allclose(y, W @ oracle.x_dec_sbvr(z, sc), rtol=1e-12, atol=1e-14)


def test_partials_identity_and_popcount():
    """O-P: element-loop counts equal popcount(beta & d) on the packed words;
    sum_j alpha_j P_tj = T_t exactly; 0 <= P <= G."""
    rng = np.random.default_rng(24)
    enc = _random_enc(rng, 4, 256, 4, 16, dyadic=False)
    x = rng.standard_normal(256).astype(np.float16)
    z, xp, sc = oracle.encode_vector(x, 128, 8)
    P, T = oracle.partials_rows(enc, z, xp)
    for r in range(4):
        for g in range(2):
            for t in range(4):
                for j in range(8):
                    pc = sum(bin(int(enc.planes[r, g, t, w]) & int(xp[g, j, w])).count("1") for w in range(4))
                    assert P[r, g, t, j] == pc
                assert int(np.dot(ALPHA8, P[r, g, t].astype(np.int64))) == T[r, g, t]
    assert P.min() >= 0 and P.max() <= 128


def test_structural_fma_count():
    """K*l coefficient products per group instead of G element FMAs (reading A13)."""
    g = json.load(open(os.path.join(GOLD, "paper_p251_fma_count.json")))
    assert g["K"] * g["l"] == g["coefficient_products_per_group"]
    assert g["element_fmas_per_group"] // g["coefficient_products_per_group"] == g["reduction_factor"]
    # the popcount form above uses exactly K*l integer partials per (row, group)
    enc = _random_enc(np.random.default_rng(25), 1, 128, g["K"], 16, dyadic=False)
    z, xp, sc = oracle.encode_vector(np.ones(128, np.float16), 128, g["l"])
    P, _ = oracle.partials_rows(enc, z, xp, l=g["l"])
    assert P[0, 0].size == g["coefficient_products_per_group"]
