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
    assert L.sbvr_abi_version() == 1
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


def test_device_layout_is_fragment_order():
    """Tile 0, lane 4*gq + c holds word c of rows gq, gq+8 for planes (0, 1): sbvr.h layout."""
    M, N, K = 16, 128, 2
    pc = np.zeros((M, 1, K, 4), np.uint32)
    for r in range(M):
        for t in range(K):
            for c in range(4):
                pc[r, 0, t, c] = (r << 16) | (t << 8) | c
    z = np.zeros((M, 1), np.uint16)
    pd = sb.pack_host(pc, z, z, z.astype(np.uint8)).view(np.uint32)
    for lane in range(32):
        gq, c = divmod(lane, 4)
        got = pd[4 * lane:4 * lane + 4].tolist()
        assert got == [(gq << 16) | c, ((gq + 8) << 16) | c, (gq << 16) | (1 << 8) | c, ((gq + 8) << 16) | (1 << 8) | c]


def test_unit_record_layout():
    """A unit = [4 tiles of planes][4 x 16 scale/bias][4 x 16 ratio index] (sbvr.h)."""
    M, N, K = 64, 256, 4
    pc = np.zeros((M, 2, K, 4), np.uint32)
    s16 = (np.arange(M * 2, dtype=np.uint16) + 1).reshape(M, 2)
    b16 = (np.arange(M * 2, dtype=np.uint16) + 1000).reshape(M, 2)
    ri = (np.arange(M * 2) % 251).astype(np.uint8).reshape(M, 2)
    data = sb.pack_host(pc, s16, b16, ri)
    ub = 4 * (256 * K + 80)
    for g in range(2):
        unit = data[g * ub:(g + 1) * ub]
        sbw = unit[4 * 256 * K:4 * 256 * K + 256].view(np.uint32)
        rib = unit[4 * 256 * K + 256:]
        for r in range(M):
            i, r16 = divmod(r, 16)
            e = 16 * i + 2 * (r16 % 8) + r16 // 8
            assert sbw[e] == (int(s16[r, g]) | (int(b16[r, g]) << 16)) and rib[e] == ri[r, g]


def test_algorithmic_bytes_match_survey_table():
    # SURVEY §8d.3 table (fp16-x path): q/o 4096x4096 K=4 -> 9,068,544 B; down 4096x14336 -> 31,698,944 B
    assert sb.algorithmic_bytes(4096, 4096, 4, act="fp16") == 9068544
    assert sb.algorithmic_bytes(4096, 14336, 4, act="fp16") == 31698944
