"""Inputs built to land EXACTLY on the real-valued ties of ⌈·⌋ (reading Q1: round half away from zero,
P:115 Eq. 2), for every quantizer on the path. Each builder returns the input and the codes the
half-away rule must produce (the half-even rule gives different codes on every constructed tie).

  * activations (O4): row max 127·2^-6 -> s_x = 2^-6 exactly; x = (j + 1/2)·2^-6
  * weights, level 1 (O1): row max 119·2^-7 -> s0 = 2^-7 exactly; W = (j + 1/2)·2^-7
  * RMSNorm -> quantize (Q23-Q25): x = ±1 everywhere (Σx²/K = 1, eps = 0 -> r = 1 exactly), so the
    fp16 layer output is γ·x and γ carries the tie grid
  * SiLU·mul -> quantize (Q24, Q26): gate = 32 (silu(32) = 32(1 - 1.3e-14), so fp16(silu·u) = 32u
    for fp16 u on the grid) and u = (j + 1/2)·2^-11"""
import numpy as np


def half_away(t):
    return np.sign(t) * np.floor(np.abs(t) + 0.5)


def tie_grid(rng, n, jmax):
    """n half-integers j + 1/2 with |j + 1/2| < jmax (both signs), as float64."""
    j = rng.integers(-jmax, jmax, n)
    return j + 0.5


def activation_rows(M, K, seed, tie_rows):
    """[M][K] fp16: rows in `tie_rows` are all exact ties (plus the max 127·2^-6); the others are
    ordinary N(0,1) rows (the division-free fast path). Returns (X, expected codes of tie rows)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((M, K)).astype(np.float16)
    want = {}
    for m in tie_rows:
        t = tie_grid(rng, K, 127)
        t[rng.integers(0, K)] = 127.0 * (1 if m % 2 else -1)
        X[m] = (t / 64).astype(np.float16)
        want[m] = half_away(t).astype(np.int64)
    return X, want


def weight_rows(N, K, seed, tie_rows):
    """[N][K] fp16 weights (N(0, 1/K)); rows in `tie_rows` are exact level-1 ties with s0 = 2^-7.
    Returns (W, expected q8 of the tie rows)."""
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float16)
    want = {}
    for n in tie_rows:
        t = tie_grid(rng, K, 119)
        t[rng.integers(0, K)] = -119.0 if n % 2 else 119.0
        W[n] = (t / 128).astype(np.float16)
        want[n] = half_away(t).astype(np.int64)
    return W, want


def rmsnorm_rows(M, K, seed):
    """(X, gamma, eps, expected codes): X = ±1, eps = 0, gamma on the 2^-6 tie grid (one row shares
    gamma, so every row's codes are ±half_away(gamma·64) by the sign of x)."""
    rng = np.random.default_rng(seed)
    X = np.where(rng.integers(0, 2, (M, K)) == 1, 1.0, -1.0).astype(np.float16)
    t = tie_grid(rng, K, 127)
    t[rng.integers(0, K)] = 127.0
    gamma = (t / 64).astype(np.float16)
    want = half_away(X.astype(np.float64) * t[None, :]).astype(np.int64)
    return X, gamma, 0.0, want


def silu_rows(M, I, seed):
    """gate_up [M][2I] fp16 = (gate = 32 | up on the 2^-11 tie grid) and the expected codes."""
    rng = np.random.default_rng(seed)
    t = np.stack([tie_grid(rng, I, 127) for _ in range(M)])
    t[np.arange(M), rng.integers(0, I, M)] = 127.0
    GU = np.empty((M, 2 * I), np.float16)
    GU[:, :I] = 32.0
    GU[:, I:] = (t / 2048).astype(np.float16)
    return GU, half_away(t).astype(np.int64)
