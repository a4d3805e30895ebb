"""Pins for the NEXT-2 oracles (activation quantization fused into RMSNorm and SiLU·mul, P:410,
Fig. 7; readings Q23-Q26 in DESIGN.md §3). Each test pins the oracle to something other
than itself: exact rational arithmetic, closed forms, invariances, scipy/numpy library routines.
CPU only (no GPU marker)."""
import math
from fractions import Fraction

import numpy as np
import pytest
import scipy.special

import oracle
import synth

# all finite non-negative fp16 values, ascending, exactly as fp64
_H = np.arange(0, 0x7c00, dtype=np.uint16).view(np.float16).astype(np.float64)


def _d2h_exact(d: float) -> int:
    """Brute-force RNE binary64 -> binary16 by exact rational comparison with the two neighbouring
    fp16 values (the definition of round-to-nearest-even, IEEE 754 §4.3.1)."""
    if d == 0.0:
        return 0x8000 if math.copysign(1.0, d) < 0 else 0
    sign = 0x8000 if d < 0 else 0
    a = abs(d)
    if a >= 65520.0:                              # >= max + half ulp (65504 + 16): overflow
        return sign | 0x7c00
    i = int(np.searchsorted(_H, a, side="right")) - 1     # _H[i] <= a < _H[i+1]
    if _H[i] == a:
        return sign | i
    lo, hi = Fraction(_H[i]), Fraction(_H[i + 1]) if i + 1 < len(_H) else Fraction(65536)
    fa = Fraction(a)
    if fa - lo < hi - fa:
        return sign | i
    if fa - lo > hi - fa:
        return sign | (i + 1)
    return sign | (i if i % 2 == 0 else i + 1)   # tie: even significand (bit 0 of the pattern)


def test_d2h_rn_matches_exact_rational_rounding():
    """Q24: one RNE rounding from fp64 — ties, ties ± 1 ulp(fp64) (which a double rounding through
    fp32 would get wrong), subnormals, the overflow boundary and random doubles."""
    rng = np.random.default_rng(7)
    mids = (_H[:-1] + _H[1:]) / 2                                   # exact in fp64
    cases = [0.0, -0.0, 2.0 ** -25, 2.0 ** -25 * 1.0000001, 2.0 ** -26, 65504.0, 65519.99, 65520.0,
             -65519.999, 1e300, 5.960464477539063e-08]
    picks = rng.choice(len(mids), 3000, replace=False)
    for m in mids[picks]:
        cases += [m, np.nextafter(m, 0.0), np.nextafter(m, np.inf), -m]
    cases += list(rng.standard_normal(2000) * 10.0 ** rng.uniform(-8, 4.5, 2000))
    for d in cases:
        assert oracle.d2h_rn(float(d)) == _d2h_exact(float(d)), d


def _exact_rinv(row_fp16: np.ndarray, eps: float) -> float:
    """Q25 independently: Python integers for Σ x²·2^48 (exact), int -> float is correctly rounded
    in Python, then IEEE fp64 (/K, +eps, math.sqrt, 1/·)."""
    S = 0
    for v in row_fp16.astype(np.float64):
        f = Fraction(float(v)) ** 2 * 2 ** 48
        assert f.denominator == 1
        S += f.numerator
    ms = math.ldexp(float(S), -48) / len(row_fp16) + eps
    return 0.0 if ms == 0.0 else 1.0 / math.sqrt(ms)


def test_rmsnorm_rinv_exact_sum_wide_dynamic_range():
    """Q25: Σx² is exact before the single fp64 rounding. Rows mixing 65504-scale and subnormal
    values (where a running fp64 sum loses the small terms) must match exact integer arithmetic."""
    rng = np.random.default_rng(3)
    naive_differs = 0
    for t in range(40):
        K = int(rng.choice([8, 128, 1000, 4096]))
        mag = 2.0 ** rng.uniform(-24, 15.9, K)
        row = (mag * rng.choice([-1, 1], K)).astype(np.float16)
        for eps in (0.0, 1e-5, 1e-6):
            r = oracle.rmsnorm_rinv(row, eps)
            assert r == _exact_rinv(row, eps), (t, K, eps)
            v = row.astype(np.float64)
            naive = float(np.sum(v * v)) / K + eps
            naive_differs += (0.0 if naive == 0 else 1.0 / math.sqrt(naive)) != r
    assert naive_differs > 0    # the rows are hard enough that summation order matters


def test_rmsnorm_constant_row_closed_form():
    """x_k = c, γ = 1, eps = 0: y = c/|c| = ±1 exactly in fp16, so q = ±127, s_x = fp16(1/127)."""
    for c in (1.0, -3.0, 0.1, 1000.0, -6.1e-5, 2.0 ** -24):
        X = np.full((1, 256), c, np.float16)
        Y = oracle.rmsnorm_fp16(X, np.ones(256, np.float16), 0.0)
        assert np.all(Y == np.float16(np.sign(c)))
        qx, sx, tx = oracle.rmsnorm_quantize(X, np.ones(256, np.float16), 0.0)
        assert np.all(qx == 127 * int(np.sign(c)))
        assert sx[0] == np.float16(np.float32(1.0) / np.float32(127.0))
        assert tx[0] == 256 * 127 * int(np.sign(c))


def test_rmsnorm_scale_invariance_and_gamma_linearity():
    """eps = 0: RMSNorm(2^j x) = RMSNorm(x) bit for bit (S scales by 4^j exactly); γ·2^j scales y by
    2^j exactly while y stays normal. A dropped 1/K, a sum of |x| instead of x², or r applied twice
    breaks one of these."""
    rng = np.random.default_rng(11)
    Z = rng.standard_normal((6, 512))
    X = (np.sign(Z) * (0.05 + np.abs(Z))).astype(np.float16)       # |x| >= 0.05: 2^-8 x stays normal
    g = (1.0 + 0.25 * rng.standard_normal(512)).astype(np.float16)
    Y = oracle.rmsnorm_fp16(X, g, 0.0)
    for j in (-8, -3, 2, 4):
        Xs = (X.astype(np.float64) * 2.0 ** j).astype(np.float16)
        assert np.array_equal(Xs.astype(np.float64), X.astype(np.float64) * 2.0 ** j)
        assert np.array_equal(oracle.rmsnorm_fp16(Xs, g, 0.0).view(np.uint16), Y.view(np.uint16))
    for j in (-2, 3):
        gs = (g.astype(np.float64) * 2.0 ** j).astype(np.float16)
        got = oracle.rmsnorm_fp16(X, gs, 0.0).astype(np.float64)
        big = np.abs(Y.astype(np.float64)) >= 2.0 ** -12
        assert np.array_equal(got[big], Y.astype(np.float64)[big] * 2.0 ** j)


def test_rmsnorm_unit_rms_and_elementwise_definition():
    """γ = 1, eps = 0: mean(y²) = 1 up to fp16 rounding; every element equals fp16((x·r)·γ) computed
    with numpy's fp64 -> fp16 conversion from the exact r; the quantized row is O4 of that output."""
    rng = np.random.default_rng(5)
    X = synth.activations_fp16(8, 4096, seed=5)
    g = (1.0 + 0.1 * rng.standard_normal(4096)).astype(np.float16)
    Y1 = oracle.rmsnorm_fp16(X, np.ones(4096, np.float16), 0.0).astype(np.float64)
    assert np.allclose(np.mean(Y1 ** 2, axis=1), 1.0, rtol=2e-3)
    eps = 1e-5
    Y = oracle.rmsnorm_fp16(X, g, eps)
    for m in range(8):
        r = _exact_rinv(X[m], eps)
        ref = np.array([_d2h_exact(float(x) * r * float(gg)) for x, gg in
                        zip(X[m].astype(np.float64), g.astype(np.float64))], np.uint16)
        assert np.array_equal(Y[m].view(np.uint16), ref), m
    qx, sx, tx = oracle.rmsnorm_quantize(X, g, eps)
    q2, s2, t2 = oracle.quantize_activations(Y)
    assert np.array_equal(qx, q2) and np.array_equal(sx, s2) and np.array_equal(tx, t2)


def test_rmsnorm_eps_and_zero_row():
    """eps enters under the square root: r = 1/sqrt(S/K + eps); an all-zero row with eps = 0 gives
    r = 0, y = 0, s_x = 1 (the Q10 all-zero rule), q = 0."""
    x = np.array([3.0, 4.0] * 64, np.float16)     # S/K = 12.5
    assert oracle.rmsnorm_rinv(x, 0.0) == 1.0 / math.sqrt(12.5)
    assert oracle.rmsnorm_rinv(x, 87.5) == 0.1
    z = np.zeros((2, 128), np.float16)
    assert oracle.rmsnorm_rinv(z[0], 0.0) == 0.0
    qx, sx, tx = oracle.rmsnorm_quantize(z, np.ones(128, np.float16), 0.0)
    assert np.all(qx == 0) and np.all(sx == 1.0) and np.all(tx == 0)


def test_rmsnorm_ldx_view_and_tail():
    """A K-view of a wider row (ldx > K) normalizes over the first K entries only."""
    X = synth.activations_fp16(3, 384, seed=9)
    g = np.ones(384, np.float16)
    a = oracle.rmsnorm_fp16(X, g, 1e-5, K=200)
    b = oracle.rmsnorm_fp16(np.ascontiguousarray(X[:, :200]), g, 1e-5)
    assert np.array_equal(a.view(np.uint16), b.view(np.uint16))


def test_silu_closed_forms():
    """silu(0) = 0; silu(x) − silu(−x) = x (σ(x) + σ(−x) = 1); silu = x·expit(x) (scipy); the
    global minimum is −W(1/e) at x = −1 − W(1/e) (W = Lambert W); silu(x) = x once e^-x < 2^-53."""
    assert oracle.silu_f64(0.0) == 0.0
    xs = np.concatenate([np.linspace(-30, 30, 1201), [1e-8, -1e-8, 65504.0 / 4096]])
    for x in xs:
        s, sm = oracle.silu_f64(x), oracle.silu_f64(-x)
        assert abs((s - sm) - x) <= 4e-16 * max(1.0, abs(x))
        assert abs(s - x * scipy.special.expit(x)) <= 4e-16 * max(1e-300, abs(s)) + 1e-300
    w = float(scipy.special.lambertw(1.0 / math.e).real)
    xmin = -1.0 - w
    assert abs(oracle.silu_f64(xmin) + w) < 1e-15
    assert oracle.silu_f64(xmin) <= min(oracle.silu_f64(xmin + d) for d in (-1e-4, 1e-4))
    assert oracle.silu_f64(40.0) == 40.0 and oracle.silu_f64(-745.0) == pytest.approx(-745.0 * math.exp(-745.0))


def test_silu_mul_elementwise_and_layouts():
    """h = fp16(silu(g)·u): u = 1 gives fp16(silu(g)); every element matches exact-rational RNE of
    the fp64 value computed with numpy's exp; the [gate | up] layout equals separate G, U; the
    quantized output is O4 of h."""
    rng = np.random.default_rng(13)
    M, K = 4, 640
    G = (rng.standard_normal((M, K)) * 3).astype(np.float16)
    U = rng.standard_normal((M, K)).astype(np.float16)
    H = oracle.silu_mul_fp16(G, U)
    g64, u64 = G.astype(np.float64), U.astype(np.float64)
    ref = np.array([[_d2h_exact(float(a / (1.0 + np.exp(-a)) * b)) for a, b in zip(gr, ur)]
                    for gr, ur in zip(g64, u64)], np.uint16)
    assert np.array_equal(H.view(np.uint16), ref)
    H1 = oracle.silu_mul_fp16(G, np.ones((M, K), np.float16))
    assert np.array_equal(H1.view(np.uint16),
                          np.array([[_d2h_exact(float(a * scipy.special.expit(a))) for a in gr] for gr in g64],
                                   np.uint16))
    GU = np.concatenate([G, U], axis=1)
    assert np.array_equal(oracle.silu_mul_fp16(GU).view(np.uint16), H.view(np.uint16))
    qx, sx, tx = oracle.silu_mul_quantize(GU)
    q2, s2, t2 = oracle.quantize_activations(H)
    assert np.array_equal(qx, q2) and np.array_equal(sx, s2) and np.array_equal(tx, t2)
