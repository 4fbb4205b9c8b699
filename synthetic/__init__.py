"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only random numbers and layer shapes.  Both the
oracle side and the CUDA side receive the same bytes from here (DESIGN.md §Input recipe).
Shapes are the public Hugging Face configs named in BASELINE.json / SURVEY.md §8d.2.
"""
from __future__ import annotations

import numpy as np
import torch

# (name, M = out_features, N = in_features)
LLAMA3_8B_LAYER = [("q_proj", 4096, 4096), ("k_proj", 1024, 4096), ("v_proj", 1024, 4096),
                   ("o_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("up_proj", 14336, 4096),
                   ("down_proj", 4096, 14336)]
LLAMA3_70B_MLP = [("down_proj", 8192, 28672), ("gate_proj", 28672, 8192), ("up_proj", 28672, 8192)]
QWEN25_7B_LAYER = [("q_proj", 3584, 3584), ("k_proj", 512, 3584), ("v_proj", 512, 3584), ("o_proj", 3584, 3584),
                   ("gate_proj", 18944, 3584), ("up_proj", 18944, 3584), ("down_proj", 3584, 18944)]


def gaussian_weight(M: int, N: int, seed: int, sigma: float = 1.0) -> np.ndarray:
    """W ~ N(0, sigma^2), float32 [M][N], torch CPU generator (SURVEY §8d.2 convention)."""
    g = torch.Generator().manual_seed(int(seed))
    return (torch.randn(M, N, generator=g, dtype=torch.float32) * sigma).numpy()


def student_t_weight(M: int, N: int, seed: int, df: float = 3.0, sigma: float = 0.02) -> np.ndarray:
    """Heavy-tailed robustness input (Student-t, df=3)."""
    rng = np.random.default_rng(seed)
    return (rng.standard_t(df, size=(M, N)) * sigma).astype(np.float32)


def hadamard_signs(N: int, seed: int) -> np.ndarray:
    """The random +-1 diagonal D of the randomized Hadamard rotation, int8 [N]."""
    rng = np.random.default_rng(seed)
    return np.where(rng.random(N) < 0.5, -1, 1).astype(np.int8)


def activation(N: int, seed: int, T: int = 1, outliers: int = 0) -> np.ndarray:
    """x ~ N(0, 1) as fp16 [T][N] (post-RMSNorm scale); optional outlier channels x50."""
    g = torch.Generator().manual_seed(int(seed))
    x = torch.randn(T, N, generator=g, dtype=torch.float32)
    if outliers:
        idx = torch.randperm(N, generator=g)[:outliers]
        x[:, idx] *= 50.0
    return x.to(torch.float16).numpy()


def with_degenerate_groups(W: np.ndarray, G: int = 128, seed: int = 0) -> np.ndarray:
    """Copy of W with a few all-zero, constant and single-outlier groups (edge cases)."""
    W = W.copy()
    M, N = W.shape
    rng = np.random.default_rng(seed)
    NG = N // G
    picks = rng.choice(M * NG, size=min(6, M * NG), replace=False)
    for k, q in enumerate(picks):
        r, g = divmod(int(q), NG)
        seg = W[r, g * G:(g + 1) * G]
        if k % 3 == 0:
            seg[:] = 0.0
        elif k % 3 == 1:
            seg[:] = np.float32(0.0123)
        else:
            seg[:] = 0.0
            seg[rng.integers(G)] = np.float32(1.5)
    return W


def random_encoded(M: int, N: int, K: int, n_ratio: int, seed: int, G: int = 128):
    """Random SBVR-encoded weights in the canonical layout (uniform bits, fp16 scale ~ |N(0.06, 0.02)|,
    fp16 bias ~ N(0, 0.003), uniform ratio index): the structure of an encoded Llama layer without
    running the (slow) encoder, for full-size GEMV parity and benchmarking."""
    rng = np.random.default_rng(seed)
    NG = N // G
    planes = rng.integers(0, 2 ** 32, size=(M, NG, K, G // 32), dtype=np.uint64).astype(np.uint32)
    s = np.abs(rng.normal(0.06, 0.02, size=(M, NG))).astype(np.float16)
    b = rng.normal(0.0, 0.003, size=(M, NG)).astype(np.float16)
    ridx = rng.integers(0, n_ratio, size=(M, NG)).astype(np.uint8)
    return planes, s.view(np.uint16), b.view(np.uint16), ridx
