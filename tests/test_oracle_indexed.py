"""Pins of the oracle's table + index storage (f2; reading A23), not re-derivations of it:

- the table entries are exactly Algorithm 1's winners of the sampled groups (re-encoded independently), distinct,
  in sample order, and the sample positions cover the matrix evenly;
- every group's index points at an entry whose MSE is the minimum over the table, found by brute force over all
  2^(K*128)-free per-element masks (each entry's MSE re-derived with numpy, independent of entry_mse);
- the bits are the nearest-subset assignment of the chosen entry (exact reconstruction check in numpy);
- when every group is sampled (n_table >= groups), each group's own winner is in the table, so the indexed MSE
  can only be lower or equal, group by group;
- the expanded (per-group) meta decodes to the same matrix as the table lookup.
"""
import itertools

import numpy as np
import pytest

import oracle
import synthetic


def _f16(h):
    return float(np.array([h], np.uint16).view(np.float16)[0])


def _np_entry_mse(X, K, r, s, b):
    """Independent numpy MSE: all 2^K subset sums, per-element minimum squared distance."""
    c = np.array([s * r ** t + b for t in range(K)])
    sums = np.array([sum(c[t] for t in range(K) if (m >> t) & 1) for m in range(1 << K)])
    return float(np.mean(np.min((X[:, None] - sums[None, :]) ** 2, axis=1)))


def test_sample_positions_even():
    for n_groups, n_table in ((64, 16), (1000, 256), (5, 16), (131072, 256)):
        pos = oracle.table_sample_positions(n_groups, n_table)
        assert len(pos) == min(n_groups, n_table)
        assert pos[0] == 0 and all(a < b for a, b in zip(pos, pos[1:])) and pos[-1] < n_groups
        gaps = np.diff(pos)
        assert gaps.size == 0 or gaps.max() - gaps.min() <= 1


@pytest.mark.parametrize("K,M,N,n_table", [(4, 8, 512, 8), (3, 16, 256, 4), (2, 4, 1024, 16)])
def test_indexed_encoding_pins(K, M, N, n_table):
    cfg = oracle.OracleConfig(K=K, n_scale=16)
    W = synthetic.with_degenerate_groups(synthetic.gaussian_weight(M, N, seed=K + M, sigma=0.02), seed=K)
    enc = oracle.encode_matrix_indexed(W, cfg, n_table)
    NG = N // 128
    R = oracle.ratio_set(cfg.n_ratio)
    # table = distinct winners of the sampled groups, in sample order
    expect = []
    for q in oracle.table_sample_positions(M * NG, n_table):
        r, g = divmod(q, NG)
        e = oracle.encode_group(W[r, 128 * g:128 * (g + 1)].astype(np.float64), cfg)
        t = (e["r_idx"], e["s16"], e["b16"])
        if t not in expect:
            expect.append(t)
    assert [tuple(int(v) for v in t) for t in enc.table] == expect
    assert enc.idx.max() < len(enc.table)
    for r in range(M):
        for g in range(NG):
            X = W[r, 128 * g:128 * (g + 1)].astype(np.float64)
            ms = [_np_entry_mse(X, K, R[ri], _f16(s), _f16(b)) for ri, s, b in enc.table]
            best = min(ms)
            assert np.isclose(enc.mse[r, g], best, rtol=1e-12, atol=1e-300)
            assert ms[enc.idx[r, g]] == pytest.approx(best, rel=1e-12, abs=1e-300)
            # bits: the reconstruction from the planes is the nearest subset sum of every element
            ri, s, b = enc.table[enc.idx[r, g]]
            c = np.array([_f16(s) * R[ri] ** t + _f16(b) for t in range(K)])
            bits = np.array([[(enc.planes[r, g, t, e // 32] >> (e % 32)) & 1 for e in range(128)] for t in range(K)])
            rec = (bits * c[:, None]).sum(0)
            sums = np.array([sum(c[t] for t in range(K) if (m >> t) & 1) for m in range(1 << K)])
            d_rec = np.abs(X - rec)
            d_min = np.min(np.abs(X[:, None] - sums[None, :]), axis=1)
            assert np.allclose(d_rec, d_min, rtol=0, atol=1e-15)


def test_all_groups_sampled_never_worse_than_full_search():
    K, M, N = 4, 4, 512
    cfg = oracle.OracleConfig(K=K, n_scale=16)
    W = synthetic.gaussian_weight(M, N, seed=3, sigma=0.02)
    full = oracle.encode_matrix(W, cfg)
    enc = oracle.encode_matrix_indexed(W, cfg, 256)                  # 16 groups, all sampled
    assert len(enc.table) <= 16
    assert np.all(enc.mse <= full.mse)


def test_expanded_meta_decodes_identically():
    K, M, N = 3, 8, 256
    cfg = oracle.OracleConfig(K=K, n_scale=16)
    enc = oracle.encode_matrix_indexed(synthetic.gaussian_weight(M, N, seed=5, sigma=0.02), cfg, 4)
    exp = enc.expand()
    D = oracle.decode_matrix(exp)
    R = oracle.ratio_set(cfg.n_ratio)
    for r, g in itertools.product(range(M), range(N // 128)):
        ri, s, b = enc.table[enc.idx[r, g]]
        c = np.array([_f16(s) * R[ri] ** t + _f16(b) for t in range(K)])
        bits = np.array([[(enc.planes[r, g, t, e // 32] >> (e % 32)) & 1 for e in range(128)] for t in range(K)])
        assert np.allclose(D[r, 128 * g:128 * (g + 1)], (bits * c[:, None]).sum(0), rtol=1e-14, atol=1e-18)
