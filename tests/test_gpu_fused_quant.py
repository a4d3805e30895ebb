"""GPU parity for activation quantization fused into RMSNorm and SiLU·mul (NEXT-2, Fig. 7
P:398-404; readings Q23-Q26) through the C ABI against the CPU oracle: q_x, s_x and t_x BIT-exact on
seeded inputs at small ragged sizes, the register path (K <= 16384), the streaming path (K > 16384),
K-views (ldx > K), degenerate rows, wide-dynamic-range rows, and the full bench sizes."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def assert_same(got, ref, what):
    qx, sx, tx = got
    q_ref, s_ref, t_ref = ref
    torch.cuda.synchronize()
    q = qx.cpu().numpy()
    bad = np.argwhere(q != q_ref)
    assert bad.size == 0, f"{what}: {len(bad)} q_x codes differ, first at {bad[:4].tolist()}"
    assert np.array_equal(sx.cpu().numpy().view(np.uint16), s_ref.view(np.uint16)), f"{what}: s_x differs"
    if tx is not None:
        assert np.array_equal(tx.cpu().numpy(), t_ref), f"{what}: t_x differs"


def hard_rows(X):
    """Degenerate / extreme rows on top of synthetic activations (where the row count allows)."""
    M, K = X.shape
    rng = np.random.default_rng(M * 7 + K)
    if M > 1:
        X[1] = 0                                                                # all-zero row
    if M > 2:
        X[2] = np.float16(0.375)                                                # constant row
    if M > 3:                                                                   # 2^-24 .. 65504 mixed
        X[3] = (2.0 ** rng.uniform(-24, 15.9, K) * rng.choice([-1, 1], K)).astype(np.float16)
    if M > 4:
        X[4] = (rng.standard_normal(K) * 1e-6).astype(np.float16)               # subnormal-heavy
    return X


RMS_SHAPES = [(1, 8), (3, 200), (16, 256), (7, 1032), (64, 4096), (5, 8192), (2, 16384),
              (3, 16392), (2, 28672)]


@pytest.mark.parametrize("M,K", RMS_SHAPES)
@pytest.mark.parametrize("eps", [1e-5, 0.0])
def test_rmsnorm_quantize_bit_exact(gpu_lib, M, K, eps):
    X = hard_rows(synth.activations_fp16(M, K, seed=M + K))
    g = synth.rmsnorm_weight_fp16(K, seed=K)
    got = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), eps)
    assert_same(got, oracle.rmsnorm_quantize(X, g, eps), f"rmsnorm M={M} K={K} eps={eps}")


@pytest.mark.parametrize("M,K,ldx", [(4, 256, 264), (6, 4096, 8192), (3, 16392, 16400)])
def test_rmsnorm_quantize_k_view(gpu_lib, M, K, ldx):
    """A K-view of wider rows (ldx > K); t_x omitted (nullable)."""
    X = synth.activations_fp16(M, ldx, seed=ldx)
    g = synth.rmsnorm_weight_fp16(K, seed=1)
    qx, sx, _ = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), 1e-5, K=K, want_tx=False)
    q_ref, s_ref, t_ref = oracle.rmsnorm_quantize(X, g, 1e-5, K=K)
    assert_same((qx, sx, None), (q_ref, s_ref, t_ref), "rmsnorm view")


def test_rmsnorm_quantize_prefill_size(gpu_lib):
    """Bench prefill size: M = 4096 tokens x K = 4096 (Llama-3-8B hidden), every code compared."""
    X = synth.activations_fp16(4096, 4096, seed=11)
    g = synth.rmsnorm_weight_fp16(4096, seed=2)
    got = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), 1e-5)
    assert_same(got, oracle.rmsnorm_quantize(X, g, 1e-5), "rmsnorm M=4096")


@pytest.mark.parametrize("K", [256, 4096, 16392])
def test_rmsnorm_exact_fp16_ties(gpu_lib, K):
    """Rows whose fp64 y lands EXACTLY on fp16 rounding midpoints (ties to even, Q24): x in {3, 1}
    with mean(x²) = 4 (r = 1/2 exactly at eps = 0) and γ = 1 + 2^-10, so y = 1.5 (1 + 2^-10) is
    1.5 ulp above 1.5 — the fp32 fast path must hand these to the exact path."""
    X = np.tile(np.array([3, 3, 3, 1, 1, 1, 1, 1], np.float16), (4, K // 8))
    X[1] *= -1
    X[2] = np.roll(X[2], 3)
    g = np.full(K, 1 + 2.0 ** -10, np.float16)
    got = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), 0.0)
    assert_same(got, oracle.rmsnorm_quantize(X, g, 0.0), f"rmsnorm ties K={K}")
    Y = oracle.rmsnorm_fp16(X, g, 0.0)
    assert Y[0, 0] == np.float16(1.5 + 2 * 2.0 ** -10)       # the tie rounded to even (up here)


SILU_SHAPES = [(1, 8), (3, 200), (16, 256), (7, 1032), (64, 14336), (2, 16384), (3, 16392), (2, 28672)]


@pytest.mark.parametrize("M,K", SILU_SHAPES)
def test_silu_mul_quantize_bit_exact(gpu_lib, M, K):
    GU = synth.gate_up_fp16(M, K, seed=M * K)
    if M > 1:
        GU[1] = 0                                                                # all-zero row
    if M > 2:                                                                    # extremes: exp over/underflow
        GU[2, :8] = np.array([65504, -65504, 40, -40, 11.09, -11.09, 1e-7, -6e-8], np.float16)
    if M > 3:                                                                    # exact fp16 ties: silu(48) = 48
        GU[3, :K] = np.float16(48.0)                                             # in fp64, 48 (1 + 2^-10) is a
        GU[3, K:] = np.float16(1 + 2.0 ** -10)                                   # midpoint (1.5 ulp above 48)
        GU[3, 1:K:2] = np.float16(-3.0)
    got = gpu_lib.silu_mul_quantize(to_dev(GU))
    assert_same(got, oracle.silu_mul_quantize(GU), f"silu M={M} K={K}")


def test_silu_mul_quantize_prefill_size(gpu_lib):
    """Bench prefill size: M = 4096 x intermediate 14336 (gate_up output [4096][28672])."""
    GU = synth.gate_up_fp16(4096, 14336, seed=5)
    got = gpu_lib.silu_mul_quantize(to_dev(GU))
    assert_same(got, oracle.silu_mul_quantize(GU), "silu M=4096")


def test_fused_equals_unfused_chain_through_gemm(gpu_lib):
    """The fused quantizer feeds the W4A8 GEMM exactly like the unfused chain (Q23): rmsnorm_quantize
    -> w4a8_gemm_i32 equals the oracle's INT32 GEMM on the oracle's quantized RMSNorm output."""
    M, N, K = 33, 384, 1024
    X = synth.activations_fp16(M, K, seed=3)
    g = synth.rmsnorm_weight_fp16(K, seed=3)
    W = synth.weights_fp16(N, K, seed=3)
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    qx, sx, tx = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), 1e-5)
    acc = gpu_lib.w4a8_gemm_i32(qx, tx, packed, N)
    torch.cuda.synchronize()
    q_ref, _, _ = oracle.rmsnorm_quantize(X, g, 1e-5)
    p_ref, _ = oracle.quantize_weights(W)
    assert np.array_equal(acc.cpu().numpy(), oracle.acc_from_packed(q_ref, p_ref, N, K))
