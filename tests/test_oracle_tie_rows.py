"""The tie-row builders (tests/tie_rows.py) against the oracle: every constructed input lands on exact
real-valued ties and the oracle's quantizers (O1, O4 and the fused RMSNorm / SiLU·mul quantizers of
Q23-Q26) produce the round-half-away codes (Q1) — so the GPU parity tests that feed the
same rows to the CUDA path compare against pinned behaviour. CPU only."""
import numpy as np

import oracle
import tie_rows


def test_activation_tie_rows_half_away():
    X, want = tie_rows.activation_rows(6, 512, seed=1, tie_rows=[0, 3, 5])
    qx, sx, tx = oracle.quantize_activations(X)
    for m, w in want.items():
        assert sx[m] == np.float16(2.0 ** -6)
        assert np.array_equal(qx[m].astype(np.int64), w)
        assert tx[m] == w.sum()


def test_weight_tie_rows_half_away():
    W, want = tie_rows.weight_rows(128, 256, seed=2, tie_rows=[1, 64, 127])
    q8, s0 = oracle.level1(W)
    for n, w in want.items():
        assert s0[n] == np.float16(2.0 ** -7)
        assert np.array_equal(q8[n].astype(np.int64), w)


def test_rmsnorm_tie_rows_half_away():
    X, g, eps, want = tie_rows.rmsnorm_rows(4, 384, seed=3)
    assert oracle.rmsnorm_rinv(X[0], eps) == 1.0
    assert np.array_equal(oracle.rmsnorm_fp16(X, g, eps), (X.astype(np.float64) * g).astype(np.float16))
    qx, sx, tx = oracle.rmsnorm_quantize(X, g, eps)
    assert np.all(sx == np.float16(2.0 ** -6))
    assert np.array_equal(qx.astype(np.int64), want)


def test_silu_tie_rows_half_away():
    GU, want = tie_rows.silu_rows(3, 256, seed=4)
    H = oracle.silu_mul_fp16(GU)
    assert np.array_equal(H.astype(np.float64), GU[:, 256:].astype(np.float64) * 32)
    qx, sx, tx = oracle.silu_mul_quantize(GU)
    assert np.all(sx == np.float16(2.0 ** -6))
    assert np.array_equal(qx.astype(np.int64), want)
