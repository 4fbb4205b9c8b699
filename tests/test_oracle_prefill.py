"""Pins of the prefill oracle O-PF (§5.1: SBVR weights decompressed into FP16, then a GEMM on
the tensor cores; reading A25 fixes how the FP16 value is formed).  Each pin ties O-PF to something other than
itself:
  * where every coefficient and every partial sum is exactly representable in fp16, the FP16 decompression must
    equal the pinned fp64 decoder (oracle.decode_matrix) exactly, and the GEMM the pinned GEMV (oracle.gemv_rows);
  * in general it must lie within the error bound of K fp16 roundings of the fp64 value, and differ from it;
  * unit-vector tokens read the decompressed weight matrix back column by column (index/transposition check);
  * the result for a batch of tokens equals the per-token results, and is linear in x.
"""
import numpy as np

import oracle
import synthetic


def _enc(M, N, K, seed, exact=False):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=seed)
    if exact:
        # r in {-1, -0.5, 0.5, 1} (ratio set endpoints, exact), s in (0, 1/2] and b in [-1/4, 1/4] multiples of
        # 2^-6: every c_t (|c_t| <= 3/4) and every partial sum of at most 4 of them (<= 3) is a multiple of 2^-9
        # below 4 in magnitude, i.e. has at most 11 significant bits: exact in fp16 (and in fp32)
        rng = np.random.default_rng(seed + 1)
        ri = rng.choice(np.array([0, 7, 8, 15], np.uint8), size=ri.shape)
        s16 = (rng.integers(1, 33, size=s16.shape) / 64.0).astype(np.float16).view(np.uint16)
        b16 = (rng.integers(-16, 17, size=b16.shape) / 64.0).astype(np.float16).view(np.uint16)
    return oracle.Encoded(M, N, oracle.OracleConfig(K=K, n_ratio=16), pc, s16, b16, ri, None)


def test_ratio_endpoints_exact():
    R = oracle.ratio_set(16)
    assert R[0] == -1.0 and R[7] == -0.5 and R[8] == 0.5 and R[15] == 1.0


def test_exact_case_equals_fp64_decoder():
    for K in (1, 2, 3, 4):
        enc = _enc(32, 256, K, seed=10 + K, exact=True)
        w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float64)
        assert np.array_equal(w16, oracle.decode_matrix(enc))


def test_exact_case_gemm_equals_gemv():
    enc = _enc(48, 384, 4, seed=21, exact=True)
    X = synthetic.activation(384, seed=22, T=3)
    Y = oracle.prefill_rows(enc, X)
    for tau in range(3):
        ref = oracle.gemv_rows(enc, oracle.x_dec_fp16(X[tau]))
        assert np.array_equal(Y[tau], ref)


def test_rounding_bound_and_not_exact():
    """|w16 - w| <= sum over the K+1 roundings (c_t to fp16, then each partial sum) of half an fp16 ulp of the
    largest magnitude involved (|c_t| and partial sums <= sum_t |c_t|), plus the fp32 error of c_t; and the FP16
    decompression really rounds (some elements differ from the fp64 decode)."""
    enc = _enc(64, 512, 4, seed=31)
    w = oracle.decode_matrix(enc)
    w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float64)
    NG = 512 // 128
    R = oracle.ratio_set(16)
    for r in range(64):
        for g in range(NG):
            c = oracle.coefficients(R[enc.r_idx[r, g]], oracle.fp16_to_double(int(enc.s16[r, g])),
                                    oracle.fp16_to_double(int(enc.b16[r, g])), 4)
            big = np.abs(c).sum()
            bound = (4 + 1) * 2.0 ** -11 * big + 4 * 2.0 ** -23 * big
            seg = slice(g * 128, (g + 1) * 128)
            assert np.abs(w16[r, seg] - w[r, seg]).max() <= bound
    assert np.count_nonzero(w16 != w) > 0.1 * w.size


def test_unit_vector_tokens_read_columns():
    enc = _enc(40, 256, 3, seed=41)
    w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float64)
    cols = [0, 1, 17, 127, 128, 200, 255]
    X = np.zeros((len(cols), 256), np.float16)
    for i, cidx in enumerate(cols):
        X[i, cidx] = 1.0
    Y = oracle.prefill_rows(enc, X)
    for i, cidx in enumerate(cols):
        assert np.array_equal(Y[i], w16[:, cidx])


def test_batch_equals_single_tokens_and_rows_subset():
    enc = _enc(64, 256, 4, seed=51)
    X = synthetic.activation(256, seed=52, T=4)
    Y = oracle.prefill_rows(enc, X)
    for tau in range(4):
        assert np.array_equal(oracle.prefill_rows(enc, X[tau:tau + 1])[0], Y[tau])
    rows = np.array([63, 0, 17, 5], np.int32)
    assert np.array_equal(oracle.prefill_rows(enc, X, rows), Y[:, rows])
    # linearity in x: doubling x (exact in fp16 and fp64) doubles y exactly
    assert np.array_equal(oracle.prefill_rows(enc, (X.astype(np.float32) * 2).astype(np.float16)), 2 * Y)


def _one_group(K, s, b, bits_per_element):
    planes = np.zeros((1, 1, K, 4), np.uint32)
    for e, bits in enumerate(bits_per_element):
        for t, bit in enumerate(bits):
            if bit:
                planes[0, 0, t, e // 32] |= np.uint32(1 << (e % 32))
    s16 = np.array([[s]], np.float16).view(np.uint16)
    b16 = np.array([[b]], np.float16).view(np.uint16)
    ri = np.array([[15]], np.uint8)                  # r = 1.0: c_t = s + b for every t
    return oracle.Encoded(1, 128, oracle.OracleConfig(K=K, n_ratio=16), planes, s16, b16, ri, None)


def test_hand_worked_rounding_examples():
    """Reading A25 by hand.  (a) s = 1 + 2^-10, b = 0, r = 1, K = 3: c16 = 1 + 2^-10 (exact); bits (1,1,1):
    fl16(2 + 2^-9) = 2 + 2^-9 (exact, ulp 2^-9 on [2, 4)), then 3 + 1.5 * 2^-9 is a tie between mantissas 513 and
    514 -> even: 3 + 2^-8 (the fp64 decode is 3 + 3 * 2^-10); bits (1,1,0) -> 2 + 2^-9; (1,0,0) -> 1 + 2^-10.
    (b) s = 1, b = 2^-12, K = 2: c32 = 1 + 2^-12 rounds to c16 = 1 (below half an ulp), so bits (1,1) give 2 while
    the fp64 decode is 2 + 2^-11."""
    enc = _one_group(3, 1.0 + 2.0 ** -10, 0.0, [(1, 1, 1), (1, 1, 0), (1, 0, 0), (0, 0, 0), (0, 1, 1)])
    w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float64)[0]
    assert list(w16[:5]) == [3 + 2.0 ** -8, 2 + 2.0 ** -9, 1 + 2.0 ** -10, 0.0, 2 + 2.0 ** -9]
    assert oracle.decode_matrix(enc)[0, 0] == 3 + 3 * 2.0 ** -10
    enc = _one_group(2, 1.0, 2.0 ** -12, [(1, 1), (0, 1)])
    w16 = oracle.prefill_decode(enc).view(np.float16).astype(np.float64)[0]
    assert list(w16[:2]) == [2.0, 1.0]
    assert oracle.decode_matrix(enc)[0, 0] == 2 + 2.0 ** -11
