"""Pins for the NEXT-4 oracles (KV4 cache and decode attention; §5.3 P:504-536, P:813;
readings Q27-Q29 in DESIGN.md §3): closed forms of softmax attention, invariances, GQA mapping, the
quantization error bound of Eq. 2 and the page layout by hand. CPU only."""
import numpy as np
import scipy.special

import oracle


def rng(seed):
    return np.random.default_rng(seed)


def test_kv4_quantize_exact_grid_and_error_bound():
    """A row on an exact grid (q - z) s reconstructs exactly; random rows reconstruct within s/2 (the
    rounding half step of Eq. 2) plus the fp16 rounding of s; the zero point is an integer in [0, 15]
    stored exactly in fp16."""
    D = 128
    g = rng(0)
    codes = g.integers(0, 16, D)
    codes[:2] = (0, 15)
    exact = ((codes - 5) * 2.0 ** -7).astype(np.float16)
    X = np.stack([exact, g.standard_normal(D).astype(np.float16), np.full(D, 0.75, np.float16)])
    q, s, z = oracle.kv4_quantize(X)
    xh = oracle.kv4_dequant(q, s, z)
    assert np.array_equal(xh[0], exact.astype(np.float64))
    zf = z.astype(np.float64)
    assert np.all(zf == np.round(zf)) and np.all((zf >= 0) & (zf <= 15))
    err = np.abs(xh[1] - X[1].astype(np.float64))
    assert err.max() <= float(s[1]) / 2 * (1 + 2 ** -9)
    assert np.all(q[2] == q[2][0])                    # constant row: one code, s = 1


def test_kv4_quantize_is_the_per_channel_rule():
    """Q27: the KV rule is the per-channel weight rule (Q20-Q22) applied per (token, head) row."""
    X = (rng(1).standard_normal((64, 128)) * 3).astype(np.float16)
    q, s, z = oracle.kv4_quantize(X)
    q2, s2, z2 = oracle.pc_quantize(X)
    assert np.array_equal(q, q2) and np.array_equal(s.view(np.uint16), s2.view(np.uint16))
    assert np.array_equal(z.astype(np.float64), z2.astype(np.float64))


def test_attention_single_token_and_uniform_keys():
    """One token: softmax of one score is 1, o = v. Equal keys: uniform weights, o = mean of v."""
    D, H = 128, 4
    Q = rng(2).standard_normal((H, D)).astype(np.float16)
    V = rng(3).standard_normal((5, 2, D))
    o = oracle.attention_f64(Q, rng(4).standard_normal((1, 2, D)), V[:1])
    assert np.allclose(o, V[0, [0, 0, 1, 1]], rtol=0, atol=1e-15)
    K = np.repeat(rng(5).standard_normal((1, 2, D)), 5, axis=0)
    o = oracle.attention_f64(Q, K, V)
    assert np.allclose(o, V.mean(axis=0)[[0, 0, 1, 1]], rtol=1e-13, atol=1e-14)


def test_attention_against_scipy_softmax_and_invariances():
    """o = softmax(q Kᵀ/√D) V against scipy.special.softmax on a small case; token permutation
    invariance; a key offset u with q·u = 0 for all heads leaves o unchanged; GQA: query head h reads kv
    head h // (H / H_kv) (§2.1)."""
    g = rng(6)
    T, H, H_kv, D = 7, 8, 2, 16
    Q = g.standard_normal((H, D)).astype(np.float16)
    K = g.standard_normal((T, H_kv, D))
    V = g.standard_normal((T, H_kv, D))
    o = oracle.attention_f64(Q, K, V)
    q64 = Q.astype(np.float64)
    for h in range(H):
        kv = h // (H // H_kv)
        p = scipy.special.softmax(K[:, kv] @ q64[h] / np.sqrt(D))
        assert np.allclose(o[h], p @ V[:, kv], rtol=1e-12, atol=1e-13)
    perm = g.permutation(T)
    assert np.allclose(oracle.attention_f64(Q, K[perm], V[perm]), o, rtol=1e-12, atol=1e-13)
    Qz = np.zeros((H, D), np.float16)
    Qz[:, : D // 2] = Q[:, : D // 2]
    u = np.zeros(D)
    u[D // 2:] = 3.0                                      # q·u = 0 for every head of Qz
    assert np.allclose(oracle.attention_f64(Qz, K + u, V), oracle.attention_f64(Qz, K, V), rtol=1e-12, atol=1e-13)


def test_attention_dominant_score_selects_its_value():
    """A key aligned with q and scaled up dominates the softmax: o -> that token's v."""
    D = 64
    Q = np.ones((1, D), np.float16)
    K = np.zeros((4, 1, D))
    K[2, 0] = 10.0
    V = rng(7).standard_normal((4, 1, D))
    assert np.allclose(oracle.attention_f64(Q, K, V)[0], V[2, 0], atol=1e-30 + 1e-12)


def test_kv4_page_layout_by_hand():
    """Q28: token t of kv head h lands in page block_table[t // P] at slot t % P; codes byte j =
    q[2j] | q[2j+1] << 4; K codes, then V codes, then K (s, z) and V (s, z) fp16 pairs."""
    T, H_kv, D, P = 5, 2, 8, 4
    g = rng(8)
    qk = g.integers(0, 16, (T, H_kv, D)).astype(np.uint8)
    qv = g.integers(0, 16, (T, H_kv, D)).astype(np.uint8)
    sk = g.random((T, H_kv)).astype(np.float16)
    zk = g.integers(0, 16, (T, H_kv)).astype(np.float16)
    sv = g.random((T, H_kv)).astype(np.float16)
    zv = g.integers(0, 16, (T, H_kv)).astype(np.float16)
    bt = np.array([2, 0], np.int32)
    pages = oracle.kv4_store((qk, sk, zk), (qv, sv, zv), bt, 3, P)
    pb = H_kv * P * (D + 8)
    assert pages.size == 3 * pb and oracle.kv4_page_bytes(H_kv, D, P) == pb
    t, h = 4, 1                                             # page bt[1] = 0, slot 0
    base = 0 * pb + h * P * (D + 8)
    assert pages[base + 0] == qk[t, h, 0] | (qk[t, h, 1] << 4)
    assert pages[base + P * D // 2 + 3] == qv[t, h, 6] | (qv[t, h, 7] << 4)
    par = pages[base + P * D: base + P * D + 16 * P // 4 * 2].view(np.uint16)
    assert par[0] == sk[t, h].view(np.uint16) and par[1] == zk[t, h].view(np.uint16)
    assert par[2 * P] == sv[t, h].view(np.uint16) and par[2 * P + 1] == zv[t, h].view(np.uint16)
    t, h = 1, 0                                             # page bt[0] = 2, slot 1
    base = 2 * pb + 1 * (D // 2)
    assert pages[base + 2] == qk[t, h, 4] | (qk[t, h, 5] << 4)
    assert np.count_nonzero(pages[pb: 2 * pb]) == 0          # page 1 is not in the table


def test_kv4_tolerance_sees_a_missing_token():
    """Negative control for the GPU attention tolerance (tests/kv4_tol.py, derived from the kernel's
    fp32 arithmetic): on the bench-shaped data (T = 1024, H = 32, H_kv = 8, an x8 outlier channel) the
    fp16-rounded exact output passes it, while the oracle with ONE token dropped fails it — for the
    last token, the first, tokens at the page and page-ring boundaries (63/64, 191/192, 383/384) and a
    seeded sample (all 1024 single-token drops fail; measured once, 2 min). Also at T = 777 (ragged)
    dropping the last token, i.e. attending over T - 1, fails it."""
    import synth
    from kv4_tol import kv4_tolerance
    D, H, H_kv = 128, 32, 8

    def rows(T, seed, scale):
        x = synth.normal(seed, 5, T * H_kv * D).reshape(T, H_kv, D) * scale
        x[:, :, 3] *= 8.0
        return x.astype(np.float16)

    for T, sample in ((1024, [0, 1, 63, 64, 191, 192, 383, 384, 1022, 1023]
                       + list(rng(11).choice(1024, 12, replace=False))), (777, [776])):
        k = oracle.kv4_quantize(rows(T, 300, 1.0).reshape(-1, D))
        v = oracle.kv4_quantize(rows(T, 400, 0.7).reshape(-1, D))
        Kh = oracle.kv4_dequant(*k).reshape(T, H_kv, D)
        Vh = oracle.kv4_dequant(*v).reshape(T, H_kv, D)
        Q = (synth.normal(9, 6, H * D).reshape(H, D) * 2.0).astype(np.float16)
        ref = oracle.attention_f64(Q, Kh, Vh)
        tol = kv4_tolerance(Q, Kh, Vh, ref)
        assert np.all(np.abs(ref.astype(np.float16).astype(np.float64) - ref) <= tol)
        old = 2e-3 * np.abs(ref) + 2e-3 * np.abs(Vh).max()                  # the round-1 bound
        assert np.median(tol) < np.median(old) / 50
        for t in sample:
            keep = np.r_[0:t, t + 1:T]
            o = oracle.attention_f64(Q, Kh[keep], Vh[keep])
            assert not np.all(np.abs(o - ref) <= tol), f"dropping token {t} of {T} passes the tolerance"
