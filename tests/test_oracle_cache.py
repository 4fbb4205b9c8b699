"""Pins of the oracle's encode-time coefficient cache (P:233 + footnote; reading A22): what the paper's
text fixes about it, checked against the oracle's own full search (which is pinned in
test_oracle_encoder.py) and against brute force."""
import itertools

import numpy as np
import pytest

import oracle
import synthetic

CFG = oracle.OracleConfig(K=3, n_ratio=4, n_scale=8, n_bias=4)


def test_cache_size_zero_is_the_full_search():
    W = synthetic.gaussian_weight(3, 512, seed=1)
    full = oracle.encode_matrix(W, CFG)
    enc, hit = oracle.encode_matrix_cached(W, CFG, cache_size=0)
    assert not hit.any()
    for a in ("planes", "s16", "b16", "r_idx", "mse"):
        assert np.array_equal(getattr(enc, a), getattr(full, a))


def test_entry_mse_is_the_brute_force_minimum_over_masks():
    X = np.random.default_rng(2).standard_normal(128)
    for r, s, b in [(-0.75, 0.6, 0.01), (0.5, 1.1, -0.2), (-1.0, 0.3, 0.0)]:
        c = np.array([s * r ** t + b for t in range(3)])
        sums = np.array([sum(c[t] for t in range(3) if (m >> t) & 1) for m in range(8)])
        ref = np.mean(np.min((X[:, None] - sums[None, :]) ** 2, axis=1))
        assert oracle.entry_mse(X, 3, r, s, b) == pytest.approx(ref, rel=1e-12)


def test_first_group_of_every_row_is_a_full_search_miss():
    W = synthetic.gaussian_weight(4, 768, seed=3)
    full = oracle.encode_matrix(W, CFG)
    enc, hit = oracle.encode_matrix_cached(W, CFG, cache_size=4)
    assert not hit[:, 0].any()
    assert np.array_equal(enc.planes[:, 0], full.planes[:, 0]) and np.array_equal(enc.mse[:, 0], full.mse[:, 0])


def test_misses_equal_the_full_search_and_hits_use_an_earlier_coefficient_set():
    W = synthetic.gaussian_weight(6, 1024, seed=4)
    full = oracle.encode_matrix(W, CFG)
    enc, hit = oracle.encode_matrix_cached(W, CFG, cache_size=4)
    R = oracle.ratio_set(CFG.n_ratio)
    for r in range(6):
        seen = []
        for g in range(8):
            trip = (enc.r_idx[r, g], enc.s16[r, g], enc.b16[r, g])
            if hit[r, g]:
                assert trip in seen                      # reused, not searched
                X = W[r, g * 128:(g + 1) * 128].astype(np.float64)
                m = oracle.entry_mse(X, 3, R[trip[0]], oracle.fp16_to_double(trip[1]), oracle.fp16_to_double(trip[2]))
                assert enc.mse[r, g] == m
                # (a cached set may even beat the group's own search: its (s, b) can lie outside the
                # group's data-derived candidate ranges S, B of Eq. 6-11)
            else:
                for a in ("planes", "s16", "b16", "r_idx", "mse"):
                    assert np.array_equal(getattr(enc, a)[r, g], getattr(full, a)[r, g])
            seen.append(trip)


def test_hit_rule_is_strictly_below_the_moving_average():
    """Row [g0, g0]: the cached set reproduces g0's MSE exactly, which is not *below* the average
    (= g0's MSE) -> miss (footnote: "below").  Row [g0, recon(g0)]: the second group is exactly
    representable by g0's set (MSE 0 < average) -> hit with MSE 0 and g0's coefficients."""
    g0 = synthetic.gaussian_weight(1, 128, seed=5)[0]
    enc0, _ = oracle.encode_matrix_cached(g0[None, :], CFG, cache_size=4)
    W = np.concatenate([g0, g0])[None, :]
    _, hit = oracle.encode_matrix_cached(W, CFG, cache_size=4)
    assert hit.tolist() == [[0, 0]]
    recon = oracle.decode_matrix(enc0)[0].astype(np.float32)
    assert np.array_equal(recon.astype(np.float64), oracle.decode_matrix(enc0)[0])   # exact in fp32
    W2 = np.concatenate([g0, recon])[None, :]
    enc2, hit2 = oracle.encode_matrix_cached(W2, CFG, cache_size=4)
    assert hit2.tolist() == [[0, 1]] and enc2.mse[0, 1] == 0.0
    assert (enc2.s16[0, 1], enc2.b16[0, 1], enc2.r_idx[0, 1]) == (enc2.s16[0, 0], enc2.b16[0, 0], enc2.r_idx[0, 0])


def test_cached_mse_stays_near_the_full_search_on_gaussian_groups():
    """SPEC S:246's acceptance guard (the paper gives no bound): mean MSE <= 1.25 x full search."""
    W = synthetic.gaussian_weight(8, 2048, seed=6)
    full = oracle.encode_matrix(W, CFG)
    enc, hit = oracle.encode_matrix_cached(W, CFG, cache_size=8)
    assert hit.mean() > 0.1
    assert enc.mse.mean() <= 1.25 * full.mse.mean()
