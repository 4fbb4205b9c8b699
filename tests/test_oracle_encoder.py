"""Pins for the encoder half of the oracle (O-W1..O-W7), independent of the oracle itself.

Each test checks the oracle against something other than its own formulas: numpy library
routines (float16 casts, percentile, linspace), brute force over masks / joint assignments /
search entries, closed forms of the representation-point cloud, and the paper's worked
example (tests/golden/).  Citations are PAPER.md lines ("P:nnn").
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ fp16 storage rounding (reading A15)
def test_fp16_rounding_matches_numpy_cast():
    rng = np.random.default_rng(0)
    mags = 10.0 ** rng.uniform(-9, 5.2, 20000)
    xs = np.concatenate([mags, -mags])
    # exact halfway cases in the normal and subnormal ranges, overflow boundary, tiny values
    q_norm = 2.0 ** -10
    q_sub = 2.0 ** -24
    xs = np.concatenate([xs, (np.arange(1, 300) + 0.5) * q_norm, (np.arange(0, 300) + 0.5) * q_sub,
                         [65504.0, 65519.99, 65520.0, 1e6, 2.0 ** -25, 3 * 2.0 ** -25, 0.0, -0.0]])
    with np.errstate(over='ignore'):
        ref = xs.astype(np.float16).view(np.uint16)
    for x, r in zip(xs, ref):
        assert oracle.fp16_bits(x) == int(r), x


def test_fp16_decode_all_patterns():
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = h.view(np.float16).astype(np.float64)
    for bits in range(0, 65536, 7):
        v = oracle.fp16_to_double(bits)
        r = ref[bits]
        if np.isnan(r):
            assert math.isnan(v)
        else:
            assert v == r and math.copysign(1, v) == math.copysign(1, r)


# ------------------------------------------------------------------ O-W1 statistics
def test_group_stats_vs_numpy():
    rng = np.random.default_rng(1)
    for _ in range(200):
        D = rng.standard_normal(128) * rng.uniform(0.01, 3)
        q95, mn, mx, mean = oracle.group_stats(D)
        assert mn == D.min() and mx == D.max()
        ref = np.percentile(D, 95)  # numpy 'linear' method == reading A6
        assert abs(q95 - ref) <= 4 * np.finfo(float).eps * (abs(D).max())
        assert abs(mean - math.fsum(D) / 128) <= 1e-15 * abs(D).max() * 4


def test_group_stats_integer_data_exact():
    D = np.random.default_rng(2).permutation(128).astype(np.float64)
    q95, mn, mx, mean = oracle.group_stats(D)
    assert (mn, mx, mean) == (0.0, 127.0, 63.5)
    assert q95 == pytest.approx(0.95 * 127, abs=1e-12)  # sorted[f] = f, so q95 = h


def test_ratio_set_is_two_linspaces():
    for n in (2, 4, 8, 16, 32):
        ref = np.concatenate([np.linspace(-1, -0.5, n // 2), np.linspace(0.5, 1, n // 2)])
        assert np.array_equal(oracle.ratio_set(n), ref)
    assert list(oracle.ratio_set(4)) == [-1.0, -0.5, 0.5, 1.0]


def _fp16(x):
    return float(np.float16(x))


def test_candidate_sets_properties():
    """Eq. 5-11, checked through properties a misreading would break."""
    rng = np.random.default_rng(3)
    cfg = oracle.OracleConfig()
    for _ in range(100):
        D = rng.standard_normal(128) * 0.02 + rng.normal() * 0.002
        R, S, B = oracle.candidates(D, cfg)
        q95 = np.percentile(D, 95)
        s_min, s_max = 2 * q95, 1.1 * (D.max() - D.min())
        assert s_max > s_min
        # S: (j+1) offsets -> first point strictly above s_min, last point == s_max (Eq. 6, 8, 11)
        assert len(S) == cfg.n_scale and np.all(np.diff(S) >= 0)
        assert S[-1] == pytest.approx(_fp16(s_max), rel=1e-3)
        assert S[0] == pytest.approx(_fp16(s_min + (s_max - s_min) / 64), rel=1e-3)
        assert S[0] > s_min * (1 - 1e-3)
        # B: b_max = 2|avg|/K, b_min = -b_max, k offsets -> includes b_min, excludes b_max (Eq. 7, 9, 10)
        bmax = 2 * abs(D.mean()) / cfg.K
        assert B[0] == pytest.approx(-bmax, rel=2e-3, abs=1e-7)
        assert B[-1] < bmax and B[-1] == pytest.approx(bmax - 2 * bmax / 16, rel=2e-3, abs=1e-7)
        assert B[8] == 0.0  # even N_bias: the middle point is exactly 0
        # candidates are exactly fp16 values (reading A15)
        for v in list(S) + list(B):
            assert _fp16(v) == v


def test_candidate_sets_degenerate_groups():
    cfg = oracle.OracleConfig()
    R, S, B = oracle.candidates(np.zeros(128), cfg)
    assert np.all(S == 0) and np.all(B == 0)
    # constant positive group: s_max clamps to 1.01 s_min (reading A18)
    R, S, B = oracle.candidates(np.full(128, 0.5), cfg)
    assert S[0] >= 1.0 and S[-1] == _fp16(1.01)
    # zero-mean group: B collapses to {0} (SPEC S:256 example)
    D = np.concatenate([np.linspace(-1, 1, 64), -np.linspace(-1, 1, 64)])
    R, S, B = oracle.candidates(D, cfg)
    assert np.all(B == 0)


# ------------------------------------------------------------------ O-W3 / O-W4 coefficients and subset sums
def test_coefficients_geometric_series():
    assert list(oracle.coefficients(0.5, 1.0, 0.0, 4)) == [1.0, 0.5, 0.25, 0.125]
    assert list(oracle.coefficients(-1.0, 2.0, 0.5, 3)) == [2.5, -1.5, 2.5]
    rng = np.random.default_rng(4)
    for _ in range(100):
        r, s, b = rng.uniform(-1, 1), rng.uniform(0, 3), rng.uniform(-0.1, 0.1)
        c = oracle.coefficients(r, s, b, 6)
        ref = s * np.power(r, np.arange(6)) + b
        assert np.allclose(c, ref, rtol=1e-14, atol=1e-15)


def test_subset_sums_brute_force():
    rng = np.random.default_rng(5)
    for K in range(1, 7):
        for _ in range(20):
            c = rng.standard_normal(K)
            v, m = oracle.subset_sums(c)
            assert sorted(m.tolist()) == list(range(1 << K))
            for vi, mi in zip(v, m):
                tot = 0.0
                for t in range(K):
                    if (mi >> t) & 1:
                        tot = tot + c[t]
                assert vi == tot
            keys = list(zip(v.tolist(), m.tolist()))
            assert keys == sorted(keys)


def test_subset_sums_paper_example_p131():
    g = _gold("paper_p131_subset_sums.json")
    rng = np.random.default_rng(6)
    for _ in range(10):
        vals = dict(zip(g["coefficients"], rng.standard_normal(3)))
        c = [vals[k] for k in g["coefficients"]]
        v, m = oracle.subset_sums(c)
        expected = sorted(sum((vals[k] for k in p), 0.0) for p in g["points"])
        assert np.allclose(sorted(v), expected, rtol=0, atol=1e-15)


def test_subset_sums_spec_example():
    g = _gold("spec_examples.json")["subset_sums"]
    v, _ = oracle.subset_sums(g["coefficients"])
    assert v.tolist() == g["sorted_values"]


def _kurtosis(v):
    v = np.asarray(v, np.float64)
    d = v - v.mean()
    return (d ** 4).mean() / (d ** 2).mean() ** 2 - 3.0


def test_representation_cloud_closed_forms():
    # r = -1/2, s = 1, b = 0, K = 4: negabinary digits -> the 16 distinct points k/8, k = -5..10
    v, _ = oracle.subset_sums(oracle.coefficients(-0.5, 1.0, 0.0, 4))
    assert v.tolist() == [k / 8 for k in range(-5, 11)]
    # r = -1: values {-2..2} with binomial multiplicities 1,4,6,4,1
    v, _ = oracle.subset_sums(oracle.coefficients(-1.0, 1.0, 0.0, 4))
    vals, counts = np.unique(v, return_counts=True)
    assert vals.tolist() == [-2, -1, 0, 1, 2] and counts.tolist() == [1, 4, 6, 4, 1]
    # Fig. 4: excess kurtosis kappa(r=-1) = -2/K, kappa(r=-0.5) = -6(n^2+1)/(5(n^2-1)), n = 2^K
    g = _gold("paper_p141_kurtosis.json")
    for K in (2, 3, 4, 6, 8):
        v1, _ = oracle.subset_sums(oracle.coefficients(-1.0, g["s"], g["b"], K))
        assert _kurtosis(v1) == pytest.approx(-2.0 / K, abs=1e-12)
        vh, _ = oracle.subset_sums(oracle.coefficients(-0.5, g["s"], g["b"], K))
        n = 2 ** K
        assert _kurtosis(vh) == pytest.approx(-6 * (n * n + 1) / (5 * (n * n - 1)), abs=1e-12)
    vh, _ = oracle.subset_sums(oracle.coefficients(-0.5, 1.0, 0.0, 8))
    assert _kurtosis(vh) == pytest.approx(g["uniform_excess_kurtosis"], abs=1e-3)


# ------------------------------------------------------------------ O-W5 nearest (Alg. 1 note 2, reading A8)
def _nearest_bisect(v, x):
    i = int(np.searchsorted(v, x, side="left"))  # first index with v >= x
    if i == 0:
        return 0
    if i == len(v):
        # leftmost index of the run of the maximum value
        j = len(v) - 1
        while j > 0 and v[j - 1] == v[j]:
            j -= 1
        return j
    lo = i - 1
    while lo > 0 and v[lo - 1] == v[lo]:
        lo -= 1
    return lo if (x - v[lo]) <= (v[i] - x) else i


def test_nearest_linear_scan_equals_bisection():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        c = rng.standard_normal(4)
        v, _ = oracle.subset_sums(c)
        for x in rng.standard_normal(4) * 2:
            a = oracle.nearest(v, x)
            b = _nearest_bisect(v, x)
            if a != b:  # only allowed when rounding makes two distances equal; then the earlier wins
                assert abs(x - v[a]) == abs(x - v[b]) and a < b
    # midpoint tie -> smaller value; duplicate value -> smaller mask
    assert oracle.nearest(np.array([0.0, 1.0]), 0.5) == 0
    v, m = oracle.subset_sums([1.0, -1.0])
    idx = oracle.nearest(v, 0.1)
    assert v[idx] == 0.0 and m[idx] == 0
    assert oracle.nearest(v, -50.0) == 0 and v[oracle.nearest(v, 50.0)] == 1.0


def test_nearest_spec_example():
    g = _gold("spec_examples.json")["nearest"]
    v, m = oracle.subset_sums(g["coefficients"])
    i = oracle.nearest(v, g["x"])
    assert v[i] == g["value"] and m[i] == sum(1 << b for b in g["mask_bits"])


def test_per_element_nearest_is_joint_optimum():
    """North star: exhaustive brute force over all 2^(K n) joint assignments on tiny groups."""
    rng = np.random.default_rng(8)
    for K in (1, 2, 3):
        for n in (1, 2, 3, 4):
            for _ in range(5):
                c = rng.standard_normal(K)
                X = rng.standard_normal(n)
                v, _ = oracle.subset_sums(c)
                sse = sum((x - v[oracle.nearest(v, x)]) ** 2 for x in X)
                pts = [sum(c[t] for t in range(K) if (mk >> t) & 1) for mk in range(1 << K)]
                best = min(sum((X[e] - pts[a[e]]) ** 2 for e in range(n))
                           for a in itertools.product(range(1 << K), repeat=n))
                assert sse == pytest.approx(best, rel=1e-12, abs=1e-15)


# ------------------------------------------------------------------ O-W6 search (Algorithm 1)
def _brute_mse(X, K, r, s, b):
    pts = np.array([sum(s * r ** t + b for t in range(K) if (mk >> t) & 1) for mk in range(1 << K)])
    return float(np.mean(np.min((X[:, None] - pts[None, :]) ** 2, axis=1)))


def test_search_finds_global_minimum_first():
    rng = np.random.default_rng(9)
    K = 3
    R = oracle.ratio_set(4)
    for _ in range(40):
        X = rng.standard_normal(32)
        S = np.sort(rng.uniform(0.5, 3, 5))
        B = rng.uniform(-0.3, 0.3, 3)
        mse, (i, j, k) = oracle.search(X, K, R, S, B)
        brute = np.array([[[_brute_mse(X, K, r, s, b) for b in B] for s in S] for r in R])
        best = brute.min()
        assert mse == pytest.approx(best, rel=1e-12)
        assert brute[i, j, k] == pytest.approx(best, rel=1e-12)
        flat = brute.reshape(-1)
        win = (i * len(S) + j) * len(B) + k
        assert np.all(flat[:win] >= mse * (1 - 1e-12))  # nothing earlier is strictly better


def test_search_representable_input_has_zero_error():
    rng = np.random.default_rng(10)
    K = 4
    R = oracle.ratio_set(8)
    for _ in range(10):
        S = np.array([_fp16(x) for x in np.sort(rng.uniform(0.1, 2, 6))])
        B = np.array([_fp16(x) for x in rng.uniform(-0.2, 0.2, 4)])
        i0, j0, k0 = rng.integers(len(R)), rng.integers(len(S)), rng.integers(len(B))
        c = oracle.coefficients(R[i0], S[j0], B[k0], K)
        v, m = oracle.subset_sums(c)
        X = v[rng.integers(0, 1 << K, 128)]
        mse, (i, j, k) = oracle.search(X, K, R, S, B)
        assert mse == 0.0
        cw = oracle.coefficients(R[i], S[j], B[k], K)
        planes = oracle.assign(X, cw)
        dec = np.array([sum(cw[t] for t in range(K) if (planes[t, e // 32] >> (e % 32)) & 1 == 1)
                        for e in range(128)])
        assert np.array_equal(dec, X)
        assert (i, j, k) <= (i0, j0, k0)  # the first zero-error entry wins


def test_encode_group_consistency_and_determinism():
    rng = np.random.default_rng(11)
    cfg = oracle.OracleConfig(n_ratio=8, n_scale=16, n_bias=8)
    for _ in range(5):
        X = rng.standard_normal(128) * 0.02
        g = oracle.encode_group(X, cfg)
        R, S, B = oracle.candidates(X, cfg)
        i, rem = divmod(g["entry"], cfg.n_scale * cfg.n_bias)
        j, k = divmod(rem, cfg.n_bias)
        assert g["r_idx"] == i and oracle.fp16_to_double(g["s16"]) == S[j] and oracle.fp16_to_double(g["b16"]) == B[k]
        c = oracle.coefficients(R[i], S[j], B[k], cfg.K)
        dec = np.array([sum((c[t] for t in range(cfg.K) if (g["planes"][t, e // 32] >> (e % 32)) & 1), 0.0)
                        for e in range(128)])
        sse = 0.0
        for e in range(128):
            sse = sse + (X[e] - dec[e]) * (X[e] - dec[e])
        assert sse / 128 == g["mse"]
        assert g["mse"] == pytest.approx(_brute_mse(X, cfg.K, R[i], S[j], B[k]), rel=1e-12)
        g2 = oracle.encode_group(X, cfg)
        assert np.array_equal(g2["planes"], g["planes"]) and g2["entry"] == g["entry"]


def test_encode_all_zero_group():
    g = oracle.encode_group(np.zeros(128), oracle.OracleConfig(n_ratio=4, n_scale=4, n_bias=4))
    assert g["mse"] == 0.0 and not g["planes"].any() and g["s16"] == 0 and g["b16"] == 0


def test_encode_matrix_thread_count_invariant():
    W = np.random.default_rng(12).standard_normal((4, 256)).astype(np.float32)
    cfg = oracle.OracleConfig(n_ratio=4, n_scale=8, n_bias=4)
    a = oracle.encode_matrix(W, cfg, nthreads=1)
    b = oracle.encode_matrix(W, cfg, nthreads=4)
    for f in ("planes", "s16", "b16", "r_idx", "mse"):
        assert np.array_equal(getattr(a, f), getattr(b, f))


def test_shannon_sanity():
    """Eq. 1: D >= sigma^2 2^(-2R); R_eff = K + 40/G bits with 5 B of metadata."""
    rng = np.random.default_rng(13)
    cfg = oracle.OracleConfig(n_ratio=8, n_scale=16, n_bias=8)
    W = rng.standard_normal((8, 128)).astype(np.float32)
    enc = oracle.encode_matrix(W, cfg)
    assert enc.mse.mean() >= 2.0 ** (-2 * (cfg.K + 40 / 128))
