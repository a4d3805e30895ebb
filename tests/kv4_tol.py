"""Derived per-element tolerance for KV4 decode attention (reading Q29).

The GPU kernel attends over the SAME dequantized cache K̂, V̂ as the oracle (pages are byte-exact and
(q - z)·s is exact in fp32), so the only differences are fp32 arithmetic and the fp16 output. Since
round 2 the kernel runs both products on tensor cores (mma.sync m16n8k16, fp32 accumulators): QK takes
fp16 q times the exact integers c - z and applies s_K·log2e/√D to the accumulator; PV takes p·s_V as a
sum of three bf16 terms (24 significant bits, i.e. the fp32 value up to ≤ u relative) times c - z. The
products are exact and every rounding is an fp32 accumulation, which the terms below bound:

  * output rounding to fp16:                       ≤ 2^-11 |o|  (+ 2^-25 absolute in the subnormal range)
  * score s_t = Σ_d q_d k̂_td / √D in fp32:        |δs_t| ≤ (D + 2)·u·S_t,  S_t = Σ_d |q_d k̂_td| / √D,
    plus the running-max subtraction:              ≤ 2u·max_t |s_t|                        (u = 2^-24)
  * exp2 (ex2.approx, ≤ 2^-22 relative) and the online-softmax / cross-warp rescales (each one more
    exp2): at most R = 64 such factors on any path, so every weight p_t carries a relative error
    ε_p ≤ max_t |δs_t| + R·2^-22; perturbing every p_t by ≤ ε_p moves o_d by ≤ 2 ε_p Σ_t p̄_t |v̂_td − o_d|
    (numerator and denominator both move)
  * Σ_t p_t v̂_td and Σ_t p_t accumulated in fp32: ≤ (T + 32)·u·Σ_t p̄_t |v̂_td| (sequential bound;
    the chunked / tree order only does better), and the final division ≤ 2u |o|.

The bound is per (head, channel): unlike a max|v̂| term, a large outlier channel does not loosen the
others. It is ~100x tighter than the round-1 bound (2e-3 |o| + 2e-3 max|v̂|), tight enough that dropping
one token of a 1024-token sequence is visible (tests/test_oracle_kv4_pins.py)."""
import numpy as np

U = 2.0 ** -24


def kv4_tolerance(Q, Khat, Vhat, ref, rescales=64):
    """Q [H][D] fp16, Khat / Vhat [T][H_kv][D] fp64 (the oracle's dequantized cache), ref [H][D] the
    fp64 oracle output -> tol [H][D]."""
    q = Q.astype(np.float64)
    H, D = q.shape
    T, H_kv, _ = Khat.shape
    R = H // H_kv
    tol = np.empty((H, D))
    for h in range(H):
        K = Khat[:, h // R, :]
        V = Vhat[:, h // R, :]
        s = K @ q[h] / np.sqrt(D)
        S = np.abs(K) @ np.abs(q[h]) / np.sqrt(D)
        p = np.exp(s - s.max())
        p /= p.sum()
        eps_p = (D + 2) * U * S.max() + 2 * U * np.abs(s).max() + rescales * 2.0 ** -22
        spread = p @ np.abs(V - ref[h][None, :])
        accum = (T + 32) * U * (p @ np.abs(V))
        tol[h] = (2.0 ** -11 + 2 * U) * np.abs(ref[h]) + 2 * eps_p * spread + accum + 2.0 ** -25
    return tol
