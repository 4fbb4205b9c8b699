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
    pb, sbb, rib, rpb = sb.weights_bytes(4096, 4096, 4)
    assert pb == 4096 * 4096 * 4 // 8 and sbb == 4096 * 32 * 4 and rib == 4096 * 32 and rpb == 16 * 4 * 4
    for M, N, K in ((4095, 4096, 4), (4096, 4000, 4), (16, 128, 9), (16, 128, 0)):
        with pytest.raises(sb.SbvrError) as e:
            sb.weights_bytes(M, N, K)
        assert e.value.status in (sb.ERR_SHAPE, sb.ERR_UNSUPPORTED)


@pytest.mark.parametrize("M,N,K", [(16, 128, 4), (80, 384, 3), (64, 256, 2), (48, 640, 1), (32, 256, 8), (208, 512, 5)])
def test_pack_unpack_roundtrip(M, N, K):
    pc, s16, b16, ri = synthetic.random_encoded(M, N, K, 16, seed=M + N + K)
    pd, sbd, rid = sb.pack_host(pc, s16, b16, ri)
    assert pd.size == M * N * K // 32
    pc2, s2, b2, r2 = sb.unpack_host(M, N, K, pd, sbd, rid)
    assert np.array_equal(pc, pc2) and np.array_equal(s16, s2) and np.array_equal(b16, b2) and np.array_equal(ri, r2)
    # every device word is written exactly once (bijection): a permutation of the canonical words
    assert np.array_equal(np.sort(pd), np.sort(pc.reshape(-1)))


def test_device_layout_is_fragment_order():
    """Tile 0, lane 4*gq + c holds word c of rows gq, gq+8 for planes (0, 1): sbvr.h layout."""
    M, N, K = 16, 128, 2
    pc = np.zeros((M, 1, K, 4), np.uint32)
    for r in range(M):
        for t in range(K):
            for c in range(4):
                pc[r, 0, t, c] = (r << 16) | (t << 8) | c
    z = np.zeros((M, 1), np.uint16)
    pd, _, _ = sb.pack_host(pc, z, z, z.astype(np.uint8))
    for lane in range(32):
        gq, c = divmod(lane, 4)
        got = pd[4 * lane:4 * lane + 4].tolist()
        assert got == [(gq << 16) | c, ((gq + 8) << 16) | c, (gq << 16) | (1 << 8) | c, ((gq + 8) << 16) | (1 << 8) | c]


def test_algorithmic_bytes_match_survey_table():
    # SURVEY §8d.3 table (fp16-x path): q/o 4096x4096 K=4 -> 9,068,544 B; down 4096x14336 -> 31,698,944 B
    assert sb.algorithmic_bytes(4096, 4096, 4, act="fp16") == 9068544
    assert sb.algorithmic_bytes(4096, 14336, 4, act="fp16") == 31698944
