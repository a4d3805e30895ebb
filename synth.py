"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no quantization, no GEMM): it only
draws numbers. It is the one module both sides may import.

Generator: a counter-based RNG — splitmix64(seed, stream, counter) -> 53-bit uniforms ->
Box-Muller normals — vectorised in numpy so any element is reproducible from
(seed, stream, index) alone.

Value recipe (SURVEY.md §8(d) "Values", mimicking the activation outliers of PAPER.md
P:300 (§4.2, "outlier channels") and P:374 (§4.3.3)):
  * weights  W ~ N(0, 1/K) in fp16, nn.Linear layout [N][K] (Q9 reading);
  * activations X ~ N(0, 1) in fp16, with n_outlier input channels (default 4, or 0.1% of K
    if larger) scaled x20, so per-token scales are outlier-dominated as in the paper.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser applied element-wise to uint64 counters."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n uniforms in (0, 1) from counters offset..offset+n-1 of (seed, stream)."""
    base = _splitmix64(np.array([(seed * 0x100000001B3 + stream) & 0xFFFFFFFFFFFFFFFF],
                                dtype=np.uint64))[0]
    ctr = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = _splitmix64(ctr ^ base) >> np.uint64(11)          # 53 random bits
    return (bits.astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, n: int) -> np.ndarray:
    """n standard normals (Box-Muller on pairs of counter-based uniforms), float64."""
    h = (n + 1) // 2
    u1 = uniform(seed, stream, h, 0)
    u2 = uniform(seed, stream, h, h)
    r = np.sqrt(-2.0 * np.log(u1))
    t = 2.0 * np.pi * u2
    return np.concatenate([r * np.cos(t), r * np.sin(t)])[:n]


def weights_fp16(N: int, K: int, seed: int = 0, std_scale: float = 1.0) -> np.ndarray:
    """W[N][K] fp16 ~ N(0, std_scale^2 / K)  (nn.Linear layout)."""
    w = normal(seed, 1, N * K) * (std_scale / np.sqrt(K))
    return w.astype(np.float16).reshape(N, K)


def outlier_channels(K: int, seed: int = 0, n_outlier: int | None = None) -> np.ndarray:
    if n_outlier is None:
        n_outlier = max(4, K // 1000)
    u = uniform(seed, 3, K)
    return np.sort(np.argsort(u)[:n_outlier])


def activations_fp16(M: int, K: int, seed: int = 0, n_outlier: int | None = None,
                     outlier_scale: float = 20.0) -> np.ndarray:
    """X[M][K] fp16 ~ N(0,1) with outlier input channels scaled by outlier_scale."""
    x = normal(seed, 2, M * K).reshape(M, K)
    if M > 0 and K > 0:
        x[:, outlier_channels(K, seed, n_outlier)] *= outlier_scale
    return x.astype(np.float16)


# Model shapes (public model configurations, not from the paper).
# Each entry: (name, N, K, kind) with kind "col" (N-sharded under TP) or "row" (K-sharded).
LLAMA3_8B = [("qkv", 6144, 4096, "col"), ("o", 4096, 4096, "row"),
             ("gate", 14336, 4096, "col"), ("up", 14336, 4096, "col"),
             ("down", 4096, 14336, "row")]
LLAMA2_70B = [("qkv", 10240, 8192, "col"), ("o", 8192, 8192, "row"),
              ("gate", 28672, 8192, "col"), ("up", 28672, 8192, "col"),
              ("down", 8192, 28672, "row")]
QWEN15_72B = [("qkv", 24576, 8192, "col"), ("o", 8192, 8192, "row"),
              ("gate", 24576, 8192, "col"), ("up", 24576, 8192, "col"),
              ("down", 8192, 24576, "row")]
MODELS = {"llama3-8b": (LLAMA3_8B, 32), "llama2-70b": (LLAMA2_70B, 80),
          "qwen1.5-72b": (QWEN15_72B, 80)}


def fuse_gate_up(shapes):
    """gate and up share their input (FFN-1, Fig. 7): serving stacks run them as
    one GEMM over the concatenated [gate; up] weight (N = 2 x intermediate). Same algorithmic bytes."""
    out = []
    for name, N, K, kind in shapes:
        if name == "gate":
            out.append(("gate_up", 2 * N, K, kind))
        elif name != "up":
            out.append((name, N, K, kind))
    return out


def rmsnorm_weight_fp16(K: int, seed: int = 0) -> np.ndarray:
    """RMSNorm gain gamma[K] fp16 ~ 1 + 0.1 N(0,1) (NEXT-2 inputs; trained gains are O(1))."""
    return (1.0 + 0.1 * normal(seed, 3, K)).astype(np.float16)


def gate_up_fp16(M: int, K: int, seed: int = 0, scale: float = 2.0) -> np.ndarray:
    """The fused gate_up GEMM output [M][2K] fp16 (gate | up) ~ N(0, scale^2): the SiLU·mul input."""
    return (normal(seed, 4, M * 2 * K).reshape(M, 2 * K) * scale).astype(np.float16)


# ---- device-side generators for the large benchmark stacks (torch's seeded Philox on the GPU;
# same distributions as above; used by bench.py only, never as oracle inputs).

def device_weights_fp16(N: int, K: int, gen, device, std_scale: float = 1.0):
    import torch
    w = torch.randn(N, K, generator=gen, device=device, dtype=torch.float32)
    return (w * (std_scale / K ** 0.5)).half()


def device_activations_fp16(M: int, K: int, gen, device, n_outlier: int | None = None,
                            outlier_scale: float = 20.0):
    import torch
    x = torch.randn(M, K, generator=gen, device=device, dtype=torch.float32)
    if M > 0 and K > 0:
        idx = torch.as_tensor(outlier_channels(K, 0, n_outlier), device=device)
        x[:, idx] *= outlier_scale
    return x.half()
