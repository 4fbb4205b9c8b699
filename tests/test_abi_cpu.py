"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/sbvr.h declares,
validates arguments, and its host layout transforms are bit-exact inverses (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2509_18172_b200 as sb
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "sbvr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sbvr_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = sb.lib()
    syms = _declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert L.sbvr_abi_version() == 2
    assert L.sbvr_status_string(2) == b"SBVR_ERR_SHAPE"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", sb.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_weights_bytes_and_validation():
    db, rpb = sb.weights_bytes(4096, 4096, 4)
    assert db == 4096 * 4096 * 4 // 8 + 5 * 4096 * 32 and rpb == 16 * 4 * 4
    assert sb.weights_bytes(80, 384, 3)[0] == 80 * 384 * 3 // 8 + 5 * 80 * 3
    for M, N, K in ((4095, 4096, 4), (4096, 4000, 4), (16, 128, 9), (16, 128, 0)):
        with pytest.raises(sb.SbvrError) as e:
            sb.weights_bytes(M, N, K)
        assert e.value.status in (sb.ERR_SHAPE, sb.ERR_UNSUPPORTED)


@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (80, 384, 3), (64, 256, 2), (48, 640, 1), (32, 256, 8), (208, 512, 5)])
def test_pack_unpack_roundtrip(M, N, K):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M + N + K)
    data = sb.pack_host(pc, s16, b16, ri)
    assert data.size == M * N * K // 8 + 5 * M * (N // 128)
    pc2, s2, b2, r2 = sb.unpack_host(M, N, K, data)
    assert np.array_equal(pc, pc2) and np.array_equal(s16, s2) and np.array_equal(b16, b2) and np.array_equal(ri, r2)
    # every byte of the packed image is written exactly once: its multiset equals the inputs' bytes
    src = np.concatenate([pc.reshape(-1).view(np.uint8), np.stack([s16, b16], -1).reshape(-1).view(np.uint8),
                          ri.reshape(-1)])
    assert np.array_equal(np.sort(data), np.sort(src))


def _swz(K, r):
    # sbvr.h: chunk t of row r is stored at chunk position t ^ swz(r)
    return {2: (r >> 2) & 1, 4: (r >> 1) & 3, 6: (r >> 2) & 1, 8: r & 7}.get(K, 0)


@pytest.mark.parametrize("K", [1, 2, 3, 4, 6, 8])
def test_device_layout_is_row_major_swizzled(K):
    """Row r of a unit holds K 16-byte plane chunks, chunk t at position t ^ swz(r) (sbvr.h)."""
    M, N = 144, 256                                  # one full 128-row block + a 16-row tail block
    pc = np.zeros((M, 2, K, 4), np.uint32)
    for r in range(M):
        for g in range(2):
            for t in range(K):
                for c in range(4):
                    pc[r, g, t, c] = (r << 12) | (g << 8) | (t << 4) | c
    z = np.zeros((M, 2), np.uint16)
    data = sb.pack_host(pc, z, z, z.astype(np.uint8))
    ub_full, ub_tail = 128 * (16 * K + 5), 16 * (16 * K + 5)
    assert data.size == 2 * ub_full + 2 * ub_tail
    for r in range(M):
        rb, rr = divmod(r, 128)
        for g in range(2):
            base = (g * ub_full) if rb == 0 else 2 * ub_full + g * ub_tail
            row = data[base + rr * 16 * K: base + (rr + 1) * 16 * K].view(np.uint32).reshape(K, 4)
            for t in range(K):
                assert row[t ^ _swz(K, rr)].tolist() == [(r << 12) | (g << 8) | (t << 4) | c for c in range(4)]


def test_swizzle_is_bank_conflict_free():
    """Eight consecutive rows' 16-byte loads of one plane chunk hit 8 distinct 16-byte bank groups."""
    for K in range(1, 9):
        for t in range(K):
            for r0 in range(0, 128, 8):
                groups = {((r * 16 * K + 16 * (t ^ _swz(K, r))) // 16) % 8 for r in range(r0, r0 + 8)}
                assert len(groups) == 8, (K, t, r0)


def test_unit_record_layout():
    """A unit = [R rows x 16K planes][R x 4 B scale/bias][R x 1 B ratio index] (sbvr.h)."""
    M, N, K = 160, 256, 4
    pc = np.zeros((M, 2, K, 4), np.uint32)
    s16 = (np.arange(M * 2, dtype=np.uint16) + 1).reshape(M, 2)
    b16 = (np.arange(M * 2, dtype=np.uint16) + 1000).reshape(M, 2)
    ri = (np.arange(M * 2) % 251).astype(np.uint8).reshape(M, 2)
    data = sb.pack_host(pc, s16, b16, ri)
    for r in range(M):
        rb, rr = divmod(r, 128)
        R = 128 if rb == 0 else M - 128
        for g in range(2):
            base = g * 128 * (16 * K + 5) if rb == 0 else 2 * 128 * (16 * K + 5) + g * R * (16 * K + 5)
            sbw = data[base + R * 16 * K: base + R * (16 * K + 4)].view(np.uint32)
            rib = data[base + R * (16 * K + 4): base + R * (16 * K + 5)]
            assert sbw[rr] == (int(s16[r, g]) | (int(b16[r, g]) << 16)) and rib[rr] == ri[r, g]


def test_algorithmic_bytes_match_survey_table():
    # SURVEY §8d.3 table (fp16-x path): q/o 4096x4096 K=4 -> 9,068,544 B; down 4096x14336 -> 31,698,944 B
    assert sb.algorithmic_bytes(4096, 4096, 4, act="fp16") == 9068544
    assert sb.algorithmic_bytes(4096, 14336, 4, act="fp16") == 31698944


@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (80, 384, 3), (208, 512, 2)])
def test_indexed_pack_unpack_roundtrip_and_size(M, N, K):
    """SBVR_META_INDEXED layout: 1 byte of meta per group (P:246 coefficient index) instead of 5."""
    pc, _, _, _ = synthetic.random_encoded(M, N, K, 16, seed=M + K)
    idx = np.random.default_rng(M).integers(0, 256, size=(M, N // 128)).astype(np.uint8)
    db, rpb, tb = sb.weights_bytes_ex(M, N, K, 16, sb.META_INDEXED)
    assert db == M * N * K // 8 + M * (N // 128) and tb == (1 + 2 * 256) * 4
    data = np.zeros(db, np.uint8)
    L = sb.lib()
    assert L.sbvr_pack_indexed(M, N, K, 128, sb._np_ptr(np.ascontiguousarray(pc)), sb._np_ptr(idx), sb._np_ptr(data)) == 0
    pc2 = np.zeros_like(pc)
    idx2 = np.zeros_like(idx)
    assert L.sbvr_unpack_indexed(M, N, K, 128, sb._np_ptr(data), sb._np_ptr(pc2), sb._np_ptr(idx2)) == 0
    assert np.array_equal(pc, pc2) and np.array_equal(idx, idx2)
    src = np.concatenate([pc.reshape(-1).view(np.uint8), idx.reshape(-1)])
    assert np.array_equal(np.sort(data), np.sort(src))
