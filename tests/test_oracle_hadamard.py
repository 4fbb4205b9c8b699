"""Pins of the oracle's randomized Hadamard rotation (§4.5, reading A21) against what the
mathematics fixes: scipy's independent Sylvester construction, orthogonality / involution, closed forms,
and the Gaussianizing effect the paper relies on (heavy tails shrink)."""
import numpy as np
import pytest
import scipy.linalg as sl
import scipy.stats as st

import oracle
import synthetic


@pytest.mark.parametrize("b", [2, 8, 32, 128, 1024])
def test_unit_signs_identity_rows_give_scipy_hadamard(b):
    """x = e_k with signs +1: the rotated rows are the columns of H_b / sqrt(b) (scipy.linalg.hadamard
    is an independent Sylvester construction)."""
    Y = oracle.hadamard_rows(np.eye(b), np.ones(b, np.int8), b)
    assert np.allclose(Y, sl.hadamard(b).T / np.sqrt(b), rtol=0, atol=1e-15)


def test_signs_multiply_columns_before_the_transform():
    b, N = 64, 256
    s = synthetic.hadamard_signs(N, seed=3)
    X = np.random.default_rng(0).standard_normal((5, N))
    H = sl.hadamard(b) / np.sqrt(b)
    ref = np.concatenate([(X[:, k * b:(k + 1) * b] * s[k * b:(k + 1) * b]) @ H.T for k in range(N // b)], axis=1)
    assert np.allclose(oracle.hadamard_rows(X, s, b), ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("b", [16, 128, 512])
def test_rotation_is_orthogonal_and_inverts(b):
    N = 4 * b
    s = synthetic.hadamard_signs(N, seed=b)
    X = np.random.default_rng(b).standard_normal((7, N))
    Y = oracle.hadamard_rows(X, s, b)
    assert np.allclose(np.linalg.norm(Y, axis=1), np.linalg.norm(X, axis=1), rtol=1e-13)
    # Q^-1 = D H / sqrt(b): H_b is symmetric and H_b H_b = b I, so transforming again with unit signs
    # and then multiplying by the signs restores X
    back = oracle.hadamard_rows(Y, np.ones(N, np.int8), b) * s
    assert np.allclose(back, X, rtol=0, atol=1e-12)


def test_unit_vector_spreads_evenly():
    b = 256
    s = synthetic.hadamard_signs(b, seed=9)
    x = np.zeros((1, b))
    x[0, 37] = 2.0
    y = oracle.hadamard_rows(x, s, b)[0]
    assert np.allclose(np.abs(y), 2.0 / np.sqrt(b), rtol=1e-14)          # one outlier -> flat vector


def test_heavy_tails_are_gaussianized():
    """The property the paper uses the rotation for: excess kurtosis of Student-t(3) rows drops
    toward the Gaussian 0 after a 128-block rotation."""
    W = synthetic.student_t_weight(64, 1024, seed=5).astype(np.float64)
    Y = oracle.hadamard_rows(W, synthetic.hadamard_signs(1024, seed=6), 128)
    k0 = st.kurtosis(W.ravel())
    k1 = st.kurtosis(Y.ravel())
    assert k0 > 3.0 and abs(k1) < 0.5 * k0 and abs(k1) < 1.5
