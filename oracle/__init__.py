"""CPU oracle for SBVR (arXiv 2509.18172) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_2509_18172_b200``) never imports it and shares no code with it.

The arithmetic lives in ``sbvr_oracle.c`` (plain fp64 C, ``-ffp-contract=off``), each
function citing the PAPER.md passage it restates.  This module only marshals numpy
arrays through ctypes and adds the numpy-level reshaping used by the tests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sbvr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, fp64, no FP contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Cfg(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int32), ("group_size", ctypes.c_int32), ("n_ratio", ctypes.c_int32),
                ("n_scale", ctypes.c_int32), ("n_bias", ctypes.c_int32), ("s_min_factor", ctypes.c_double)]


@dataclass(frozen=True)
class OracleConfig:
    """Encoder knobs: K, group size, N_ratio/N_scale/N_bias (reading A4),
    s_min factor (P:187 = 2.0; reading A1)."""
    K: int = 4
    group_size: int = 128
    n_ratio: int = 16
    n_scale: int = 64
    n_bias: int = 16
    s_min_factor: float = 2.0

    def c(self) -> _Cfg:
        return _Cfg(self.K, self.group_size, self.n_ratio, self.n_scale, self.n_bias, self.s_min_factor)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, f64 = ctypes.c_int32, ctypes.c_double
        L.oracle_fp16_bits.restype = ctypes.c_uint16
        L.oracle_fp16_bits.argtypes = [f64]
        L.oracle_fp16_to_double.restype = f64
        L.oracle_fp16_to_double.argtypes = [ctypes.c_uint16]
        L.oracle_group_stats.argtypes = [P, i32, P, P, P, P]
        L.oracle_ratio_set.argtypes = [i32, P]
        L.oracle_candidates.argtypes = [P, i32, ctypes.POINTER(_Cfg), P, P, P]
        L.oracle_coefficients.argtypes = [f64, f64, f64, i32, P]
        L.oracle_subset_sums.argtypes = [P, i32, P, P]
        L.oracle_nearest.restype = i32
        L.oracle_nearest.argtypes = [P, i32, f64]
        L.oracle_search.restype = f64
        L.oracle_search.argtypes = [P, i32, i32, P, i32, P, i32, P, i32, P, P, P]
        L.oracle_assign.argtypes = [P, i32, P, i32, P]
        L.oracle_encode_group.restype = f64
        L.oracle_encode_group.argtypes = [P, ctypes.POINTER(_Cfg), P, P, P, P, P]
        L.oracle_encode_matrix.restype = i32
        L.oracle_encode_matrix.argtypes = [P, i32, i32, ctypes.POINTER(_Cfg), P, P, P, P, P, i32]
        L.oracle_encode_vector.argtypes = [P, i32, i32, i32, P, P, P]
        L.oracle_decode_matrix.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, P]
        L.oracle_gemv_rows.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, P, P, i32, P]
        L.oracle_partials_rows.argtypes = [P, P, P, i32, i32, i32, i32, P, i32, P, P]
        L.oracle_max_threads.restype = i32
        L.oracle_hadamard_rows.argtypes = [P, P, i32, i32, i32, P]
        L.oracle_prefill_decode_fp16.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, P]
        L.oracle_prefill_rows.argtypes = [P, P, P, P, i32, i32, i32, i32, i32, P, i32, P, i32, P]
        L.oracle_entry_mse.restype = f64
        L.oracle_entry_mse.argtypes = [P, i32, i32, f64, f64, f64]
        L.oracle_encode_matrix_cached.restype = i32
        L.oracle_encode_matrix_cached.argtypes = [P, i32, i32, ctypes.POINTER(_Cfg), i32, f64, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------------ scalar helpers
def fp16_bits(x: float) -> int:
    return int(lib().oracle_fp16_bits(float(x)))


def fp16_to_double(h: int) -> float:
    return float(lib().oracle_fp16_to_double(int(h)))


def group_stats(D):
    D = np.ascontiguousarray(D, dtype=np.float64)
    out = [ctypes.c_double() for _ in range(4)]
    lib().oracle_group_stats(_p(D), len(D), *[ctypes.byref(o) for o in out])
    return tuple(o.value for o in out)  # q95, min, max, mean


def ratio_set(n_ratio: int) -> np.ndarray:
    R = np.zeros(n_ratio, np.float64)
    lib().oracle_ratio_set(n_ratio, _p(R))
    return R


def candidates(D, cfg: OracleConfig):
    D = np.ascontiguousarray(D, dtype=np.float64)
    R = np.zeros(cfg.n_ratio, np.float64)
    S = np.zeros(cfg.n_scale, np.float64)
    B = np.zeros(cfg.n_bias, np.float64)
    c = cfg.c()
    lib().oracle_candidates(_p(D), len(D), ctypes.byref(c), _p(R), _p(S), _p(B))
    return R, S, B


def coefficients(r: float, s: float, b: float, K: int) -> np.ndarray:
    c = np.zeros(K, np.float64)
    lib().oracle_coefficients(float(r), float(s), float(b), K, _p(c))
    return c


def subset_sums(c):
    c = np.ascontiguousarray(c, dtype=np.float64)
    K = len(c)
    v = np.zeros(1 << K, np.float64)
    m = np.zeros(1 << K, np.int32)
    lib().oracle_subset_sums(_p(c), K, _p(v), _p(m))
    return v, m


def nearest(v_sorted, x: float) -> int:
    v = np.ascontiguousarray(v_sorted, dtype=np.float64)
    return int(lib().oracle_nearest(_p(v), len(v), float(x)))


def search(X, K: int, R, S, B):
    """Algorithm 1 over an explicit search space R x S x B. Returns (mse, (i, j, k))."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    R = np.ascontiguousarray(R, dtype=np.float64)
    S = np.ascontiguousarray(S, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    bi, bj, bk = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    mse = lib().oracle_search(_p(X), len(X), K, _p(R), len(R), _p(S), len(S), _p(B), len(B), ctypes.byref(bi),
                              ctypes.byref(bj), ctypes.byref(bk))
    return mse, (bi.value, bj.value, bk.value)


def assign(X, c):
    """P:231 bit assignment: planes [K][n/32] for coefficients c."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    assert len(X) % 32 == 0
    planes = np.zeros((len(c), len(X) // 32), np.uint32)
    lib().oracle_assign(_p(X), len(X), _p(c), len(c), _p(planes))
    return planes


def encode_group(X, cfg: OracleConfig):
    X = np.ascontiguousarray(X, dtype=np.float64)
    assert len(X) == cfg.group_size
    planes = np.zeros((cfg.K, cfg.group_size // 32), np.uint32)
    s16 = ctypes.c_uint16()
    b16 = ctypes.c_uint16()
    ridx = ctypes.c_uint8()
    entry = ctypes.c_int32()
    c = cfg.c()
    mse = lib().oracle_encode_group(_p(X), ctypes.byref(c), _p(planes), ctypes.byref(s16), ctypes.byref(b16),
                                    ctypes.byref(ridx), ctypes.byref(entry))
    return dict(planes=planes, s16=s16.value, b16=b16.value, r_idx=ridx.value, entry=entry.value, mse=mse)


@dataclass
class Encoded:
    """Oracle-side encoded matrix in the canonical interchange layout."""
    M: int
    N: int
    cfg: OracleConfig
    planes: np.ndarray   # [M][N/G][K][G/32] uint32
    s16: np.ndarray      # [M][N/G] uint16 (fp16 bits)
    b16: np.ndarray      # [M][N/G] uint16
    r_idx: np.ndarray    # [M][N/G] uint8
    mse: np.ndarray      # [M][N/G] float64
    threads: int = 1


def encode_matrix(W, cfg: OracleConfig, nthreads: int = 0) -> Encoded:
    W = np.ascontiguousarray(W, dtype=np.float32)
    M, N = W.shape
    G = cfg.group_size
    assert N % G == 0
    NG = N // G
    planes = np.zeros((M, NG, cfg.K, G // 32), np.uint32)
    s16 = np.zeros((M, NG), np.uint16)
    b16 = np.zeros((M, NG), np.uint16)
    ridx = np.zeros((M, NG), np.uint8)
    mse = np.zeros((M, NG), np.float64)
    c = cfg.c()
    used = lib().oracle_encode_matrix(_p(W), M, N, ctypes.byref(c), _p(planes), _p(s16), _p(b16), _p(ridx),
                                      _p(mse), int(nthreads))
    return Encoded(M, N, cfg, planes, s16, b16, ridx, mse, used)


def encode_vector(x16, G: int = 128, l: int = 8):
    """O-X: returns z [N] int32, planes [N/G][l][G/32] uint32, scales [N/G] float32."""
    x16 = np.ascontiguousarray(x16, dtype=np.float16)
    N = x16.shape[0]
    z = np.zeros(N, np.int32)
    planes = np.zeros((N // G, l, G // 32), np.uint32)
    scales = np.zeros(N // G, np.float32)
    lib().oracle_encode_vector(_p(x16.view(np.uint16)), N, G, l, _p(z), _p(planes), _p(scales))
    return z, planes, scales


def decode_matrix(enc: Encoded) -> np.ndarray:
    W = np.zeros((enc.M, enc.N), np.float64)
    lib().oracle_decode_matrix(_p(enc.planes), _p(enc.s16), _p(enc.b16), _p(enc.r_idx), enc.M, enc.N, enc.cfg.K,
                               enc.cfg.group_size, enc.cfg.n_ratio, _p(W))
    return W


def gemv_rows(enc: Encoded, x_dec, rows=None) -> np.ndarray:
    """O-Y: y_r = sum_c w_dec[r,c] x_dec[c] in fp64 for the requested rows."""
    x_dec = np.ascontiguousarray(x_dec, dtype=np.float64)
    rows = np.arange(enc.M, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    y = np.zeros(len(rows), np.float64)
    lib().oracle_gemv_rows(_p(enc.planes), _p(enc.s16), _p(enc.b16), _p(enc.r_idx), enc.M, enc.N, enc.cfg.K,
                           enc.cfg.group_size, enc.cfg.n_ratio, _p(x_dec), _p(rows), len(rows), _p(y))
    return y


def prefill_decode(enc: Encoded) -> np.ndarray:
    """O-PF decode (§5.1, reading A25): the FP16 decompressed weights [M][N] as uint16 bit patterns."""
    W16 = np.zeros((enc.M, enc.N), np.uint16)
    lib().oracle_prefill_decode_fp16(_p(enc.planes), _p(enc.s16), _p(enc.b16), _p(enc.r_idx), enc.M, enc.N,
                                     enc.cfg.K, enc.cfg.group_size, enc.cfg.n_ratio, _p(W16))
    return W16


def prefill_rows(enc: Encoded, X16, rows=None) -> np.ndarray:
    """O-PF GEMM: Y[tau][i] = sum_e w16[rows[i], e] x16[tau, e] in fp64; X16 fp16 [T][N]."""
    X16 = np.ascontiguousarray(np.asarray(X16, np.float16).reshape(-1, enc.N)).view(np.uint16)
    rows = np.arange(enc.M, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    T = X16.shape[0]
    Y = np.zeros((T, len(rows)), np.float64)
    lib().oracle_prefill_rows(_p(enc.planes), _p(enc.s16), _p(enc.b16), _p(enc.r_idx), enc.M, enc.N, enc.cfg.K,
                              enc.cfg.group_size, enc.cfg.n_ratio, _p(X16), T, _p(rows), len(rows), _p(Y))
    return Y


def x_dec_fp16(x16) -> np.ndarray:
    """fp16-x path: x_dec = fp64(x) (exact)."""
    return np.asarray(x16, dtype=np.float16).astype(np.float64)


def x_dec_sbvr(z, scales, G: int = 128) -> np.ndarray:
    """SBVR-x path: x_dec[e] = z[e] * s_x[group(e)] (exact in fp64)."""
    return np.asarray(z, np.float64) * np.repeat(np.asarray(scales, np.float64), G)


def partials_rows(enc: Encoded, z, xplanes, l: int = 8, rows=None):
    """O-P: P [rows][N/G][K][l] and T [rows][N/G][K] (element loops, not popcount)."""
    rows = np.arange(enc.M, dtype=np.int32) if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    NG = enc.N // enc.cfg.group_size
    P = np.zeros((len(rows), NG, enc.cfg.K, l), np.int32)
    T = np.zeros((len(rows), NG, enc.cfg.K), np.int32)
    z = np.ascontiguousarray(z, dtype=np.int32)
    xplanes = np.ascontiguousarray(xplanes, dtype=np.uint32)
    lib().oracle_partials_rows(_p(enc.planes), _p(z), _p(xplanes), enc.N, enc.cfg.K, enc.cfg.group_size, l, _p(rows),
                               len(rows), _p(P), _p(T))
    return P, T


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def hadamard_rows(X, signs, b: int) -> np.ndarray:
    """Randomized block Hadamard rotation along N (§4.5; reading A21): every block of b columns
    of every row becomes H_b diag(signs) x / sqrt(b), fp64, plain O(b^2) definition."""
    X = np.ascontiguousarray(np.asarray(X, np.float64))
    rows, N = X.shape
    assert N % b == 0 and b & (b - 1) == 0
    sg = np.ascontiguousarray(np.asarray(signs, np.int8))
    assert sg.shape == (N,)
    Y = np.empty_like(X)
    lib().oracle_hadamard_rows(_p(X), _p(Y), rows, N, b, _p(sg))
    return Y


def entry_mse(X, K: int, r: float, s: float, b: float) -> float:
    """MSE of one group under the coefficient set c_t = s r^t + b (Eq. 4) with nearest-subset-sum
    assignment -- the quantity Algorithm 1 minimises."""
    X = np.ascontiguousarray(np.asarray(X, np.float64))
    return lib().oracle_entry_mse(_p(X), X.size, K, float(r), float(s), float(b))


def encode_matrix_cached(W, cfg: OracleConfig, cache_size: int = 8, alpha: float = 0.1):
    """Encode with the encode-time coefficient cache (P:233 + footnote; reading A22): per row, groups
    left to right, MRU cache of (r, s, b), hit when the best cached MSE < the moving average.
    Returns (Encoded, hit[M][NG] uint8)."""
    W = np.ascontiguousarray(np.asarray(W, np.float32))
    M, N = W.shape
    G, K = cfg.group_size, cfg.K
    NG = N // G
    planes = np.zeros((M, NG, K, G // 32), np.uint32)
    s16 = np.zeros((M, NG), np.uint16)
    b16 = np.zeros((M, NG), np.uint16)
    ri = np.zeros((M, NG), np.uint8)
    mse = np.zeros((M, NG), np.float64)
    hit = np.zeros((M, NG), np.uint8)
    c = cfg.c()
    lib().oracle_encode_matrix_cached(_p(W), M, N, ctypes.byref(c), int(cache_size), float(alpha), _p(planes), _p(s16),
                                      _p(b16), _p(ri), _p(mse), _p(hit))
    return Encoded(M, N, cfg, planes, s16, b16, ri, mse), hit



# ------------------------------------------------------------------ coefficient table + per-group index (f2)
def table_sample_positions(n_groups: int, n_table: int):
    """Reading A23: the coefficient table is seeded from min(n_table, n_groups) evenly spaced groups,
    q_i = floor(i * n_groups / n_sample) in row-major (row, group) order."""
    n_s = min(n_table, n_groups)
    return [i * n_groups // n_s for i in range(n_s)]


@dataclass
class IndexedEncoded:
    """SBVR weights in the table + index format: planes as Encoded, a coefficient table of
    (r_idx, s16, b16) entries and one u8 table index per group."""
    M: int
    N: int
    cfg: OracleConfig
    planes: np.ndarray   # [M][N/G][K][G/32] uint32
    idx: np.ndarray      # [M][N/G] uint8
    table: np.ndarray    # [n][3] (r_idx, s16, b16) as int64
    mse: np.ndarray      # [M][N/G] float64

    def expand(self) -> Encoded:
        """The per-group meta the table entries stand for (same decode, the plain format)."""
        t = self.table[self.idx.astype(np.int64)]
        return Encoded(self.M, self.N, self.cfg, self.planes, t[..., 1].astype(np.uint16), t[..., 2].astype(np.uint16),
                       t[..., 0].astype(np.uint8), self.mse)


def encode_matrix_indexed(W, cfg: OracleConfig, n_table: int) -> IndexedEncoded:
    """f2 storage ("a coefficient cache containing all coefficient sets required for decoding, as well as a
    coefficient index that identifies the specific coefficient set used by each K-bit bitvector set"; P:233 the
    cache of previously selected r, s, b), reading A23, step by step:
      1. Algorithm 1 (encode_group) on the table_sample_positions groups;
      2. the table = their winning (r_idx, s16, b16) triples, duplicates dropped, in sample order (<= n_table <= 256);
      3. every group takes the table entry of least MSE (entry_mse, strict '<' in table order: the first best) and
         its bits are assigned for that entry's coefficients."""
    W = np.ascontiguousarray(np.asarray(W, np.float32))
    M, N = W.shape
    G, K = cfg.group_size, cfg.K
    NG = N // G
    assert 1 <= n_table <= 256
    table = []
    for q in table_sample_positions(M * NG, n_table):
        r, g = divmod(q, NG)
        e = encode_group(W[r, g * G:(g + 1) * G].astype(np.float64), cfg)
        t = (int(e["r_idx"]), int(e["s16"]), int(e["b16"]))
        if t not in table:
            table.append(t)
    R = ratio_set(cfg.n_ratio)
    planes = np.zeros((M, NG, K, G // 32), np.uint32)
    idx = np.zeros((M, NG), np.uint8)
    mse = np.zeros((M, NG), np.float64)
    for r in range(M):
        for g in range(NG):
            X = W[r, g * G:(g + 1) * G].astype(np.float64)
            best, best_m = 0, None
            for e, (ri, s16, b16) in enumerate(table):
                m = entry_mse(X, K, R[ri], fp16_to_double(s16), fp16_to_double(b16))
                if best_m is None or m < best_m:
                    best, best_m = e, m
            ri, s16, b16 = table[best]
            planes[r, g] = assign(X, coefficients(R[ri], fp16_to_double(s16), fp16_to_double(b16), K))
            idx[r, g] = best
            mse[r, g] = best_m
    return IndexedEncoded(M, N, cfg, planes, idx, np.asarray(table, np.int64).reshape(-1, 3), mse)
