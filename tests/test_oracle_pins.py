"""Pins for the CPU oracle (oracle/), checked against what the paper and mathematics fix — not
against the oracle itself. Each test names the passage or property it pins.
CPU only (no GPU marker)."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ fp16 conversions (Q8/Q10)

def test_h2f_all_fp16_vs_numpy():
    """h2f against numpy's independent binary16 decoder, all 65536 patterns."""
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    ref = bits.view(np.float16).astype(np.float32)
    got = np.array([oracle.h2f(int(b)) for b in bits], np.float32)
    fin = np.isfinite(ref)
    assert np.array_equal(got[fin].view(np.uint32), ref[fin].view(np.uint32))
    assert np.all(np.isnan(got[np.isnan(ref)]))
    assert np.array_equal(got[np.isinf(ref)], ref[np.isinf(ref)])


def test_f2h_rn_vs_numpy_ties_and_random():
    """f2h_rn (RNE) against numpy's independent fp32->fp16 rounding: every fp16 value, every
    midpoint between consecutive finite fp16 values (the ties), and random fp32 bit patterns."""
    h = np.arange(0, 0x7c00, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = ((h[:-1] + h[1:]) / 2).astype(np.float32)          # exact in fp32
    rng = np.random.default_rng(0)
    rnd = rng.integers(0, 2**32, 60000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    rnd = rnd[np.isfinite(rnd)]
    xs = np.concatenate([h.astype(np.float32), mids, -mids[::7], rnd,
                         np.array([65504, 65519.99, 65520, 1e-8, 2.0**-25, 2.0**-24 * 1.5],
                                  np.float32)])
    with np.errstate(over="ignore"):
        ref = xs.astype(np.float16).view(np.uint16)
    got = np.array([oracle.f2h_rn(float(x)) for x in xs], np.uint16)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (xs[bad[:5]], got[bad[:5]], ref[bad[:5]])


def test_rhai_is_round_half_away():
    """Q1: ⌈a/b⌋ with ties away from zero, against exact rationals."""
    for b in range(1, 20):
        for a in range(-300, 301):
            f = Fraction(a, b)
            fl = f.numerator // f.denominator
            frac = f - fl
            if frac > Fraction(1, 2) or (frac == Fraction(1, 2) and f > 0):
                want = fl + 1
            else:
                want = fl
            assert oracle.rhai(a, b) == want, (a, b)


# ------------------------------------------------------------------ level 2

def _group_with(lo, hi, extra=(), g=128):
    v = [lo, hi, *extra]
    v += [lo] * (g - len(v))
    return np.array(v, np.int8)


def test_level2_paper_example_p257_overflows():
    """P:257 worked example: [-113,120] -> s=16, z=7, code(120)=15, dequant 128 > 127.
    Negative control: it also rules out round-half-to-even (⌈7.5+7⌋ would be 14)."""
    ex = gold("p257_overflow_example.json")
    qu4, s, z = oracle.level2_group(_group_with(ex["group_lo"], ex["group_hi"]))
    assert (s, z) == (ex["s_u8"], ex["z"])
    assert qu4[1] == ex["code_of_hi"]
    assert (int(qu4[1]) - z) * s == ex["qhat_of_hi"]


def test_level2_hand_worked_protective_group():
    ex = gold("protective_group.json")
    vals = [int(k) for k in ex["codes"]]
    qu4, s, z = oracle.level2_group(_group_with(ex["lo"], ex["hi"], vals))
    assert (s, z) == (ex["s_u8"], ex["z"])
    for i, v in enumerate(vals):
        assert qu4[2 + i] == ex["codes"][str(v)]
        assert (int(qu4[2 + i]) - z) * s == ex["qhat"][str(v)]


def _exhaustive(R):
    """Every reachable (lo, hi, q) with -R <= lo <= q <= hi <= R: one group per (lo, hi) holding
    lo, hi and every q between them (g = 2R+2)."""
    g = 2 * R + 2
    rows = []
    for lo in range(-R, R + 1):
        for hi in range(lo, R + 1):
            v = list(range(lo, hi + 1))
            v += [lo] * (g - len(v))
            rows.append(v)
    q8 = np.array(rows, np.int8)
    qu4, s, z = oracle.level2(q8, g)
    qhat = oracle.dequant_level2(qu4, s, z, g)
    return q8, qu4, s, z, qhat


def test_protective_range_exhaustive_119():
    """with level-1 codes in [-119,119], every reachable dequantized q̂ fits INT8
    (SURVEY PROBE-B: 0 violations, q̂ in [-121,126], max s_u8 = 16 — tighter than P:267's 17)."""
    q8, qu4, s, z, qhat = _exhaustive(119)
    assert qhat.min() >= -128 and qhat.max() <= 127
    assert qhat.min() == -121 and qhat.max() == 126
    assert s.max() == 16 and s.min() >= 1
    assert z.max() <= 15 and qu4.max() <= 15
    # z*s_u8 fits the u8 zs byte of the packed tile (north_star "precomputed z*s_u8")
    assert (z.astype(int) * s.astype(int)).max() <= 126
    # Eq. 3 reconstruction error for groups straddling 0 (lo <= 0 <= hi; the all-positive /
    # all-negative corner of Q4 is excluded): s/2 from rounding, plus at most 15/2 because the
    # integer scale ⌈(hi-lo)/15⌋ can round down, so 15 s >= (hi - lo) - 7.5 and the
    # [0,15] code clamp may bind at one end. Most codes stay within s/2.
    lo, hi = q8.min(axis=1), q8.max(axis=1)
    st = (lo <= 0) & (hi >= 0)
    err = np.abs(qhat.astype(int) - q8.astype(int))[st]
    sst = s[st].astype(int)
    assert np.all(2 * err <= sst + 15)
    assert np.mean(2 * err <= sst) > 0.95


def test_protective_range_120_is_not_safe():
    """P:267-275 derive 119.5 as the bound: one more level (R=120) already overflows. SURVEY
    PROBE-B (an independent exact-integer enumeration) counted exactly 7 overflowing triples."""
    q8, qu4, s, z, qhat = _exhaustive(120)
    bad = set()
    for r in range(q8.shape[0]):
        for i in np.nonzero((qhat[r] > 127) | (qhat[r] < -128))[0]:
            bad.add((int(q8[r].min()), int(q8[r].max()), int(q8[r, i])))
    assert len(bad) == 7


def test_level2_degenerate_and_single_value_groups():
    """Q3: a constant group gives s = 1; it must reconstruct exactly when z fits u4."""
    for v in (-119, -15, -3, 0, 5, 119):
        qu4, s, z = oracle.level2_group(np.full(128, v, np.int8))
        assert s == 1
        q = (qu4.astype(int) - z) * s
        if -15 <= v <= 0:
            assert np.all(q == v)
        # always inside INT8
        assert q.min() >= -128 and q.max() <= 127


# ------------------------------------------------------------------ level 1

def test_level1_exact_multiples_reproduce():
    """Special case: W = s0 * q with q integers in [-119,119] and s0 = 2^-7 quantizes exactly."""
    rng = np.random.default_rng(1)
    q = rng.integers(-119, 120, (4, 256))
    q[:, 0] = 119
    q[1, 0] = -119
    W = (q / 128.0).astype(np.float16)
    q8, s0 = oracle.level1(W)
    assert np.all(s0 == np.float16(2.0 ** -7))
    assert np.array_equal(q8.astype(int), q)


def test_level1_bounds_and_special_rows():
    W = synth.weights_fp16(64, 512, seed=3)
    W[1] = 0
    W[2, :] = np.float16(1e-7)         # s0 underflows -> 2^-24 rule (Q8)
    q8, s0 = oracle.level1(W)
    Wf = W.astype(np.float64)
    s = s0.astype(np.float64)
    assert s0[1] == np.float16(1.0) and np.all(q8[1] == 0)
    assert s0[2].view(np.uint16) == 1
    assert np.all(np.abs(q8) <= 119)
    normal = np.array([i not in (1, 2) for i in range(64)])
    err = np.abs(Wf - q8 * s[:, None])[normal]
    assert np.all(err <= s[normal, None] / 2 * (1 + 1e-6))
    # each row's largest-magnitude weight lands on the edge of the protective range
    assert np.all(np.abs(q8[normal]).max(axis=1) == 119)


def test_level1_scale_rule_all_fp16_amax():
    """Scale rule over every positive finite fp16 row max (SURVEY PROBE-I, an independent numpy
    sweep): the 59 row maxima with amax/119 <= 2^-25 (fp16 underflow) take the 2^-24 rule, the
    ±119 clamp engages (|W|/s0 >= 119.5) for 1687, and the largest |W|/s0 with a normal s0
    is 119.0557."""
    a = np.arange(1, 0x7c00, dtype=np.uint16).view(np.float16)
    W = a.reshape(-1, 1)
    q8, s0 = oracle.level1(W)
    sb = s0.view(np.uint16)
    under = a.astype(np.float64) / 119 <= 2.0 ** -25
    assert int(under.sum()) == 59 and np.all(sb[under] == 1)
    ratio = a.astype(np.float64) / s0.astype(np.float64)
    assert int((ratio >= 119.5).sum()) == 1687
    norm = sb >= 0x0400
    assert abs(ratio[norm].max() - 119.0557) < 1e-3
    assert np.all(np.abs(q8) <= 119)


# ------------------------------------------------------------------ activations

def test_activations_exact_multiples_zero_row_and_sums():
    rng = np.random.default_rng(2)
    q = rng.integers(-127, 128, (5, 384))
    q[:, 7] = 127
    X = (q / 64.0).astype(np.float16)      # s_x = 127/64/127 = 2^-6 exactly
    X[3] = 0
    qx, sx, tx = oracle.quantize_activations(X)
    for m in (0, 1, 2, 4):
        assert sx[m] == np.float16(2.0 ** -6)
        assert np.array_equal(qx[m].astype(int), q[m])
    assert sx[3] == np.float16(1.0) and np.all(qx[3] == 0)
    assert np.array_equal(tx, qx.astype(np.int64).sum(axis=1))


def test_activations_bounds_ldx_and_scale_rule():
    X = synth.activations_fp16(33, 700, seed=4)
    qx, sx, tx = oracle.quantize_activations(X, K=640)   # a K-view of a wider row (ldx = 700)
    Xf = X[:, :640].astype(np.float64)
    s = sx.astype(np.float64)
    assert np.all(np.abs(Xf - qx * s[:, None]) <= s[:, None] / 2 * (1 + 1e-6))
    assert np.all(np.abs(qx).max(axis=1) == 127)
    a = np.arange(1, 0x7c00, dtype=np.uint16).view(np.float16).reshape(-1, 1)
    q, sxa, _ = oracle.quantize_activations(a)
    under = a[:, 0].astype(np.float64) / 127 <= 2.0 ** -25         # PROBE-I: 63 underflows
    assert int(under.sum()) == 63 and np.all(sxa.view(np.uint16)[under] == 1)
    ratio = a[:, 0].astype(np.float64) / sxa.astype(np.float64)
    assert int((ratio >= 127.5).sum()) == 1772                     # clamp engages for 1772
    assert np.all(np.abs(q) <= 127)


# ------------------------------------------------------------------ pack

def test_pack_rlp_word_matches_paper_interleave():
    """Fig. 9 / P:447 interleave w0,w16,w1,w17,... and the SPEC S:336 word 0x76543210."""
    ex = gold("rlp_word.json")
    qu4 = np.zeros((128, 128), np.uint8)
    qu4[0, 0:4] = ex["weights_w0_w1_w2_w3"]
    qu4[0, 16:20] = ex["weights_w16_w17_w18_w19"]
    s = np.ones((128, 1), np.uint8)
    z = np.zeros((128, 1), np.uint8)
    p = oracle.pack(qu4, s, z)
    word = int.from_bytes(bytes(p[0:4]), "little")
    assert word == int(ex["word_le_u32"], 16)
    assert [(word >> (8 * i)) & 15 for i in range(4)] == ex["low_nibble_lanes"]
    assert [(word >> (8 * i + 4)) & 15 for i in range(4)] == ex["high_nibble_lanes"]


def test_pack_layout_bytes_by_hand_and_roundtrip():
    N, K = 256, 384
    rng = np.random.default_rng(5)
    qu4 = rng.integers(0, 16, (N, K)).astype(np.uint8)
    s = rng.integers(1, 17, (N, K // 128)).astype(np.uint8)
    z = rng.integers(0, 8, (N, K // 128)).astype(np.uint8)
    p = oracle.pack(qu4, s, z)
    assert p.size == 2 * 3 * 8448
    # tile (nt=1, j=2), row r=5, chunk c=3, byte b=9 <-> k = 256 + 96 + 9 and k + 16
    t = (1 * 3 + 2) * 8448
    n, k = 128 + 5, 256 + 96 + 9
    assert p[t + 3 * 2048 + 5 * 16 + 9] == qu4[n, k] | (qu4[n, k + 16] << 4)
    assert p[t + 8192 + 5] == s[n, 2]
    assert p[t + 8320 + 5] == z[n, 2] * s[n, 2]
    u, su, zu = oracle.unpack(p, N, K)
    assert np.array_equal(u, qu4) and np.array_equal(su, s) and np.array_equal(zu, z)


def test_pack_rejects_bad_shapes():
    with pytest.raises(ValueError):
        oracle.pack(np.zeros((100, 128), np.uint8), np.ones((100, 1), np.uint8),
                    np.zeros((100, 1), np.uint8))


# ------------------------------------------------------------------ GEMM and epilogue

def test_gemm_i32_matches_numpy_int64_and_detects_overflow():
    rng = np.random.default_rng(6)
    qx = rng.integers(-127, 128, (7, 300)).astype(np.int8)
    qh = rng.integers(-121, 127, (9, 300)).astype(np.int16)
    acc = oracle.gemm_i32(qx, qh)
    assert np.array_equal(acc, qx.astype(np.int64) @ qh.astype(np.int64).T)
    big_x = np.full((1, 140000), 127, np.int8)
    big_w = np.full((1, 140000), 126, np.int16)
    with pytest.raises(ValueError):
        oracle.gemm_i32(big_x, big_w)


def test_epilogue_fp64_is_exact_and_equals_bruteforce():
    """Σ_k (q_x s_x)(q̂ s0) in fp64 equals acc·s_x·s0 exactly in any order."""
    X = synth.activations_fp16(5, 256, seed=7)
    W = synth.weights_fp16(128, 256, seed=7)
    packed, s0 = oracle.quantize_weights(W)
    qx, sx, _ = oracle.quantize_activations(X)
    qu4, s, z = oracle.unpack(packed, 128, 256)
    qh = oracle.dequant_level2(qu4, s, z)
    acc = oracle.gemm_i32(qx, qh)
    y = oracle.epilogue_f64(acc, sx, s0)
    xs = qx.astype(np.float64) * sx.astype(np.float64)[:, None]
    ws = qh.astype(np.float64) * s0.astype(np.float64)[:, None]
    for m in range(5):
        for n in range(0, 128, 17):
            terms = xs[m] * ws[n]
            assert float(np.sum(terms)) == y[m, n]
            assert float(np.sum(terms[::-1])) == y[m, n]
            assert Fraction(y[m, n]) == Fraction(int(acc[m, n])) * Fraction(float(sx[m])) \
                * Fraction(float(s0[n]))


def test_hand_worked_end_to_end():
    ex = gold("hand_worked_e2e.json")
    K = ex["K"]
    W = np.zeros((128, K), np.float16)
    W[0, :3] = ex["w_first3"]
    X = np.zeros((1, K), np.float16)
    X[0, :3] = ex["x_first3"]
    q8, s0 = oracle.level1(W)
    assert float(s0[0]) == ex["s0"] and list(q8[0, :3]) == ex["q8_first3"]
    qu4, s, z = oracle.level2(q8)
    assert (s[0, 0], z[0, 0]) == (ex["s_u8"], ex["z"])
    assert list(qu4[0, :3]) == ex["qu4_first3"] and np.all(qu4[0, 3:] == ex["qu4_of_zero"])
    packed = oracle.pack(qu4, s, z)
    assert packed[8320] == ex["zs"]
    qx, sx, _ = oracle.quantize_activations(X)
    assert float(sx[0]) == ex["s_x"] and list(qx[0, :3]) == ex["qx_first3"]
    acc = oracle.acc_from_packed(qx, packed, 128, K)
    assert acc[0, 0] == ex["acc"]
    y = oracle.linear_rows(X, packed, s0, 128)
    assert abs(y[0, 0] - ex["y_exact"]) < 1e-15
    assert float(np.float16(y[0, 0])) == ex["y_fp16"]


def test_w4a8_reduces_to_float_gemm_with_bounded_error():
    """Sanity envelope (not parity): vs the unquantized float GEMM the relative Frobenius error
    on config 1 with 4 outlier channels is about 0.10-0.12 (SURVEY PROBE-F)."""
    X = synth.activations_fp16(16, 256, seed=0)
    W = synth.weights_fp16(256, 256, seed=0)
    packed, s0 = oracle.quantize_weights(W)
    y = oracle.linear_rows(X, packed, s0, 256)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert 0.01 < rel < 0.2


def test_linear_rows_subset_equals_full():
    X = synth.activations_fp16(9, 256, seed=8)
    W = synth.weights_fp16(128, 256, seed=8)
    packed, s0 = oracle.quantize_weights(W)
    full = oracle.linear_rows(X, packed, s0, 128)
    part = oracle.linear_rows(X, packed, s0, 128, 3, 7)
    assert np.array_equal(full[3:7], part)


# ------------------------------------------------------------------ NEXT-1: per-channel W4A8 (§5.2.2)

def test_pc_quantize_exact_grid_reproduces():
    """Eq. 2 on rows that ARE an asymmetric u4 grid: W = (q - z) * s with s a power of
    two and every code 0..15 present, so min/max give range = 15 s exactly. PC1 must recover s, z
    and every q (the closed form; any sign / offset / rounding slip breaks it)."""
    rng = np.random.default_rng(11)
    N, K = 6, 64
    s_true = [2.0 ** -6, 2.0 ** -3, 0.5, 2.0 ** -10, 1.0, 2.0 ** -4]
    z_true = [7, 0, 15, 3, 9, 12]
    q_true = rng.integers(0, 16, size=(N, K))
    q_true[:, 0], q_true[:, 1] = 0, 15                      # min and max codes present
    W = ((q_true - np.array(z_true)[:, None]) * np.array(s_true)[:, None]).astype(np.float16)
    qu4, s, z = oracle.pc_quantize(W)
    assert np.array_equal(s.astype(np.float64), np.array(s_true))
    assert list(z) == z_true
    assert np.array_equal(qu4, q_true)


def test_pc_quantize_bounds_and_invariants():
    """Every code in [0, 15], z in [0, 15]; when the rounded code is not clamped the dequantized
    weight (q - z) s is within s/2 of W (round-to-nearest of Eq. 2); the row's min and max map to
    the end codes up to one step (the zero point absorbs the offset)."""
    W = synth.weights_fp16(64, 512, seed=3)
    qu4, s, z = oracle.pc_quantize(W)
    assert qu4.min() >= 0 and qu4.max() <= 15 and z.max() <= 15
    sd = s.astype(np.float64)[:, None]
    Wd = W.astype(np.float64)
    t = Wd / sd + z[:, None]
    inside = (t > -0.5) & (t < 15.5)
    err = np.abs(Wd - (qu4.astype(np.float64) - z[:, None]) * sd)
    assert np.all(err[inside] <= sd.repeat(W.shape[1], 1)[inside] / 2 * (1 + 2e-6))
    assert np.all(qu4.min(1) <= 1) and np.all(qu4.max(1) >= 14)


def test_pc_quantize_half_away_ties_and_degenerate_rows():
    """Q1 in Eq. 2: a weight exactly half a step off the grid rounds AWAY from zero in t + z
    (t + z = 2.5 -> 3, not 2 as half-even or half-down would give); a constant row has range 0 ->
    s = 1 (Q20) and codes from z = ⌈-min⌋ clamped; an all-zero row quantizes to z = 0, q = 0."""
    s_ = 2.0 ** -4
    row = np.array([0, 15, 4.5, 0.5, 1.5, 7.5], np.float64)       # codes offset by z = 0 -> t + z
    W = np.zeros((3, 128), np.float16)
    W[0, :6] = (row * s_).astype(np.float16)
    W[0, 6:] = 0
    W[1, :] = np.float16(0.25)
    qu4, s, z = oracle.pc_quantize(W)
    assert float(s[0]) == s_ and z[0] == 0
    assert list(qu4[0, :6]) == [0, 15, 5, 1, 2, 8]                # 4.5 -> 5, 0.5 -> 1, 7.5 -> 8
    assert float(s[1]) == 1.0 and z[1] == 0 and np.all(qu4[1] == 0)   # ⌈0.25⌋ = 0
    assert float(s[2]) == 1.0 and z[2] == 0 and np.all(qu4[2] == 0)


def test_pc_pack_is_the_o3_nibble_stream_and_roundtrips():
    """The per-channel tile is byte-for-byte the first 8192 bytes of the pinned O3 tile for the
    same codes (P:447 interleave, Q15), and pc_unpack inverts pc_pack."""
    rng = np.random.default_rng(5)
    N, K = 256, 384
    q = rng.integers(0, 16, size=(N, K)).astype(np.uint8)
    pc = oracle.pc_pack(q)
    o3 = oracle.pack(q, np.ones((N, K // 128), np.uint8), np.zeros((N, K // 128), np.uint8))
    tiles_pc = pc.reshape(-1, 8192)
    tiles_o3 = o3.reshape(-1, 8448)[:, :8192]
    assert np.array_equal(tiles_pc, tiles_o3)
    assert np.array_equal(oracle.pc_unpack(pc, N, K), q)


def test_pc_gemm_equals_subtraction_after_multiplication():
    """Eq. (per_channel_qmm_step2/3) P:466-478 in integers: sum_k qx (q - z) == (Q_X Q_W) - z t_X
    with t_X = sum_k qx (the exact form of the paper's t_X, Q19). The right side is computed with
    the pinned O5 GEMM on q as-is and the pinned O4 row sums — a different route from PC's
    definition — and must agree exactly; int32 overflow is detected."""
    X = synth.activations_fp16(16, 256, seed=9)
    W = synth.weights_fp16(128, 256, seed=9)
    qx, sx, tx = oracle.quantize_activations(X)
    qu4, s, z = oracle.pc_quantize(W)
    acc = oracle.pc_gemm_i32(qx, qu4, z)
    rhs = oracle.gemm_i32(qx, qu4.astype(np.int16)).astype(np.int64) - np.outer(tx, z.astype(np.int64))
    assert np.array_equal(acc.astype(np.int64), rhs)
    big = np.full((1, 1200000), 127, np.int8)           # 127 * 15 * 1.2e6 > 2^31
    with pytest.raises(ValueError):
        oracle.pc_gemm_i32(big, np.full((1, 1200000), 15, np.uint8), np.zeros(1, np.uint8))


def test_pc_linear_approximates_float_gemm():
    """Sanity envelope (not parity): per-channel W4A8 of a float GEMM, y = acc s_x s_w, is within a
    few tens of percent (relative Frobenius) of the unquantized product — 4-bit per-channel weights
    are coarser than the g128 path but still track it."""
    X = synth.activations_fp16(16, 512, seed=1)
    W = synth.weights_fp16(256, 512, seed=1)
    qx, sx, tx = oracle.quantize_activations(X)
    qu4, s, z = oracle.pc_quantize(W)
    y = oracle.epilogue_f64(oracle.pc_gemm_i32(qx, qu4, z), sx, s)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    rel = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert 0.02 < rel < 0.35, rel


# ------------------------------------------------------------------ Q1 tie rule

def test_level1_real_valued_ties_round_half_away():
    """Q1 (Eq. 2 P:115 ⌈·⌋; P:257's ⌈120/16 + 7⌋ = 15 rules out half-even): level 1 rounds an
    exact half AWAY from zero. The row max 119·2^-7 gives s0 = 2^-7 exactly, so W = (k + 1/2)·2^-7
    lands on W/s0 = k + 0.5 in fp32 with no rounding: 2.5 -> 3 (half-even 2), -2.5 -> -3,
    0.5 -> 1 (half-even 0), -0.5 -> -1, 1.5 -> 2, 118.5 -> 119."""
    halves = np.array([2.5, -2.5, 0.5, -0.5, 1.5, -1.5, 118.5, -118.5, 3.5, 4.5])
    W = np.zeros((1, 128), np.float16)
    W[0, 0] = 119 / 128
    W[0, 1:1 + len(halves)] = (halves / 128).astype(np.float16)
    assert np.array_equal(W[0, 1:1 + len(halves)].astype(np.float64) * 128, halves)   # exact in fp16
    q8, s0 = oracle.level1(W)
    assert s0[0] == np.float16(2.0 ** -7)
    assert list(q8[0, 1:1 + len(halves)]) == [3, -3, 1, -1, 2, -2, 119, -119, 4, 5]


def test_activations_real_valued_ties_round_half_away():
    """Q1 for O4: with the row max 127·2^-6 the scale is s_x = 2^-6 exactly and
    x = (k + 1/2)·2^-6 gives x/s_x = k + 0.5: 2.5 -> 3, -2.5 -> -3, 0.5 -> 1, 126.5 -> 127; t_x
    sums the half-away codes."""
    halves = np.array([2.5, -2.5, 0.5, -0.5, 126.5, -126.5, 5.5, -7.5])
    X = np.zeros((2, 256), np.float16)
    X[:, 0] = 127 / 64
    X[0, 1:1 + len(halves)] = (halves / 64).astype(np.float16)
    X[1, 100:100 + len(halves)] = (-halves / 64).astype(np.float16)
    qx, sx, tx = oracle.quantize_activations(X)
    want = [3, -3, 1, -1, 127, -127, 6, -8]
    assert np.all(sx == np.float16(2.0 ** -6))
    assert list(qx[0, 1:1 + len(halves)]) == want
    assert list(qx[1, 100:100 + len(halves)]) == [-w for w in want]
    assert list(tx) == [127 + sum(want), 127 - sum(want)]
