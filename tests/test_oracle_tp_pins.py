"""Pins of oracle.tp_reduce_rank_order (NEXT-3's reduction; reading Q32: fp16 partials summed in fp32 in rank
order, one rounding to fp16) against values fixed by IEEE arithmetic, not by the oracle itself."""
from fractions import Fraction

import numpy as np
import pytest

import oracle


def f16(x):
    return np.float16(x)


def test_single_rank_is_identity_on_every_fp16():
    """R = 1: fp16 -> fp32 -> fp16 is exact for every finite fp16 (the fused kernel at world 1 equals the GEMM)."""
    bits = np.arange(0, 1 << 16, dtype=np.uint32).astype(np.uint16)
    v = bits.view(np.float16)
    v = v[np.isfinite(v)]
    out = oracle.tp_reduce_rank_order([v])
    assert np.array_equal(out.view(np.uint16), v.view(np.uint16))


@pytest.mark.parametrize("R", [2, 3, 4, 8])
def test_exact_when_fp32_sums_are_exact(R):
    """Partials with |y| in [1, 256) are multiples of 2^-10 below 2^8, so any sum of <= 8 of them is a multiple of
    2^-10 below 2^11: at most 21 significant bits, exact in fp32. The result is then the correctly rounded fp16
    of the exact rational sum (computed with Fractions)."""
    rng = np.random.default_rng(R)
    Y = [f16(rng.uniform(1.0, 255.0, size=257) * rng.choice([-1.0, 1.0], size=257)) for _ in range(R)]
    out = oracle.tp_reduce_rank_order(Y)
    for i in range(257):
        exact = sum(Fraction(float(y[i])) for y in Y)
        # exact rational -> fp16 by RNE: float(exact) is exact here (<= 22 bits), then numpy's RNE to fp16
        assert float(exact) == exact
        assert out[i].view(np.uint16) == np.float16(float(exact)).view(np.uint16), i


def test_rank_order_is_sequential_not_reversed_or_pairwise():
    """fp32 absorption (ulp(32768) = 2^-8 in fp32) makes the order observable: sequential rank order gives
    [32768, -32768, s] -> s, while reversed order gives 0; [32768, s, -32768, s] -> s sequentially but 0 as a
    pairwise tree ((32768 + s) + (-32768 + s)). s = 2^-10 (a normal fp16)."""
    s = f16(2.0 ** -10)
    big = f16(32768.0)
    one = lambda *v: [np.array([x], np.float16) for x in v]
    assert oracle.tp_reduce_rank_order(one(big, -big, s))[0] == s
    assert oracle.tp_reduce_rank_order(one(s, big, -big))[0] == 0      # s absorbed first
    assert oracle.tp_reduce_rank_order(one(big, s, -big, s))[0] == s   # a pairwise tree would give 0


def test_within_north_star_tolerance_of_fp64_sum():
    """The single fp16 rounding of an fp32 sum of <= 8 fp16 partials of one sign-mixed row stays within the
    north_star's |err| <= 2e-3 |ref| + 1e-3 of the exact fp64 sum."""
    rng = np.random.default_rng(7)
    Y = [f16(rng.normal(0, 4, size=4096)) for _ in range(8)]
    out = oracle.tp_reduce_rank_order(Y).astype(np.float64)
    ref = np.sum([y.astype(np.float64) for y in Y], axis=0)
    assert np.all(np.abs(out - ref) <= 2e-3 * np.abs(ref) + 1e-3)
