"""GPU parity holes closed in round 2 ("Next round" item 1):

* exact real-valued ties (reading Q1, round half away) through every quantizer on the
  CUDA path: the per-token quantizer (quant8's exact near-tie branch and its division-free fast path on
  the same launch), the weight packer (level2_pack_kernel's level-1 codes), the fused-prologue linear
  (qoq_w4a8_linear with QOQ_LINEAR_FUSED=1) and the fused RMSNorm / SiLU·mul quantizers (NEXT-2);
* the prefill regime M >= 1024 (north_star: >= 70% of the INT8 peak there) on all four Llama-3-8B
  projections at M = 1024, 2048, 4096 with the planner's token tile AND each of BN = 128 / 192 / 256
  forced (QOQ_BN_BIG): the 2 x 192-column TMEM accumulator stages, the single-stage 256 tile and the
  band-major work order (down_proj, K = 14336: MB < MT) all run here. INT32 accumulators bit-exact and
  Y within the north_star tolerance on sampled token rows that hit every token tile; plus per-channel
  W4A8 (NEXT-1) at M = 4096.

Inputs: tests/tie_rows.py (its oracle pins: tests/test_oracle_tie_rows.py) and synth.py."""
import functools

import numpy as np
import pytest
import torch

import oracle
import synth
import tie_rows

pytestmark = pytest.mark.gpu
RTOL, ATOL = 2e-3, 1e-3


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def bits16(t):
    return t.cpu().numpy().view(np.uint16)


def check_y(y, y_ref):
    y = np.asarray(y, np.float64)
    err = np.abs(y - y_ref)
    bad = err > RTOL * np.abs(y_ref) + ATOL
    assert not bad.any(), f"{bad.sum()} outputs outside tolerance; max err {err.max()}"


# ------------------------------------------------------------------ exact ties (Q1)

@pytest.mark.parametrize("M,K", [(8, 128), (8, 4096), (5, 14336), (70, 1024)])
def test_quantize_activations_exact_ties(gpu_lib, M, K):
    X, want = tie_rows.activation_rows(M, K, seed=K + M, tie_rows=[0, 2, M - 1])
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    assert np.array_equal(bits16(sx), sx_ref.view(np.uint16))
    assert np.array_equal(qx.cpu().numpy(), qx_ref)
    assert np.array_equal(tx.cpu().numpy(), tx_ref)
    for m, w in want.items():
        assert np.array_equal(qx[m].cpu().numpy().astype(np.int64), w)


@pytest.mark.parametrize("N,K", [(256, 512), (1280, 4096)])
def test_quantize_weights_exact_ties(gpu_lib, N, K):
    W, want = tie_rows.weight_rows(N, K, seed=N, tie_rows=[0, 1, 130, N - 1])
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    p_ref, s0_ref = oracle.quantize_weights(W)
    assert np.array_equal(bits16(s0), s0_ref.view(np.uint16))
    assert np.array_equal(packed.cpu().numpy(), p_ref)
    q8, _ = oracle.level1(W)
    for n, w in want.items():
        assert np.array_equal(q8[n].astype(np.int64), w)


@pytest.mark.parametrize("path", ["fused", "two"])
@pytest.mark.parametrize("M,N,K", [(16, 256, 1024), (64, 4096, 4096)])
def test_linear_prologue_exact_ties(gpu_lib, monkeypatch, path, M, N, K):
    """qoq_w4a8_linear on tie rows: the q_x / s_x / t_x it leaves in its workspace (the fused GEMM
    prologue's own quantization when QOQ_LINEAR_FUSED=1) are bit-exact, and Y matches the oracle."""
    if path == "fused":
        monkeypatch.setenv("QOQ_LINEAR_FUSED", "1")
    else:
        monkeypatch.delenv("QOQ_LINEAR_FUSED", raising=False)
    X, want = tie_rows.activation_rows(M, K, seed=M + K, tie_rows=[0, 3, M - 1])
    W = synth.weights_fp16(N, K, seed=3)
    p_ref, s0_ref = oracle.quantize_weights(W)
    ws = torch.zeros(gpu_lib.linear_workspace_bytes(M, N, K), dtype=torch.uint8, device="cuda:0")

    class _WS:
        def get(self, n):
            return ws, ws.numel()

    Y = gpu_lib.w4a8_linear(to_dev(X), to_dev(p_ref), to_dev(s0_ref), N, K, workspace=_WS())
    torch.cuda.synchronize()
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    qx, sx, tx = gpu_lib.linear_workspace_views(ws, M, N, K)
    assert np.array_equal(qx.cpu().numpy(), qx_ref)
    assert np.array_equal(bits16(sx), sx_ref.view(np.uint16))
    assert np.array_equal(tx.cpu().numpy(), tx_ref)
    check_y(Y.cpu().numpy(), oracle.epilogue_f64(oracle.acc_from_packed(qx_ref, p_ref, N, K), sx_ref, s0_ref))


@pytest.mark.parametrize("M,K", [(4, 4096), (64, 1024)])
def test_rmsnorm_quantize_exact_ties(gpu_lib, M, K):
    X, g, eps, want = tie_rows.rmsnorm_rows(M, K, seed=K)
    qx, sx, tx = gpu_lib.rmsnorm_quantize(to_dev(X), to_dev(g), eps)
    ref = oracle.rmsnorm_quantize(X, g, eps)
    assert np.array_equal(qx.cpu().numpy(), ref[0])
    assert np.array_equal(bits16(sx), ref[1].view(np.uint16))
    assert np.array_equal(tx.cpu().numpy(), ref[2])
    assert np.array_equal(qx.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("M,I", [(4, 14336), (64, 1024)])
def test_silu_mul_quantize_exact_ties(gpu_lib, M, I):
    GU, want = tie_rows.silu_rows(M, I, seed=I)
    qx, sx, tx = gpu_lib.silu_mul_quantize(to_dev(GU))
    ref = oracle.silu_mul_quantize(GU)
    assert np.array_equal(qx.cpu().numpy(), ref[0])
    assert np.array_equal(bits16(sx), ref[1].view(np.uint16))
    assert np.array_equal(tx.cpu().numpy(), ref[2])
    assert np.array_equal(qx.cpu().numpy().astype(np.int64), want)


# ------------------------------------------------------------------ prefill sizes (M >= 1024)

PREFILL_SHAPES = [(n, N, K) for n, N, K, _ in synth.fuse_gate_up(synth.LLAMA3_8B)]


@functools.lru_cache(maxsize=1)
def _weights(N, K):
    W = synth.weights_fp16(N, K, seed=N + 7 * K)
    p_ref, s0_ref = oracle.quantize_weights(W)
    qu4, s, z = oracle.unpack(p_ref, N, K)
    return p_ref, s0_ref, oracle.dequant_level2(qu4, s, z), to_dev(p_ref), to_dev(s0_ref)


@functools.lru_cache(maxsize=2)
def _acts(M, K):
    X = synth.activations_fp16(M, K, seed=M + K)
    return X, to_dev(X)


def sample_rows(M):
    """One row in every 64-token block (so every token tile of any BN >= 64 is hit, at a varying
    offset inside it) plus the last row."""
    return sorted({64 * i + (37 * i) % 64 for i in range(M // 64)} | {M - 1})


PREFILL_CASES = [(name, N, K, M, bn) for name, N, K in PREFILL_SHAPES for M in (1024, 2048, 4096)
                 for bn in ("auto", "128", "192", "256")]


@pytest.mark.parametrize("name,N,K,M,bn", PREFILL_CASES)
def test_prefill_gemm_sampled_bit_exact(gpu_lib, monkeypatch, name, N, K, M, bn):
    if bn == "auto":
        monkeypatch.delenv("QOQ_BN_BIG", raising=False)
    else:
        monkeypatch.setenv("QOQ_BN_BIG", bn)
    p_ref, s0_ref, qhat, packed, s0 = _weights(N, K)
    X, Xd = _acts(M, K)
    qx, sx, tx = gpu_lib.quantize_activations_per_token(Xd)
    ws = gpu_lib.Workspace(torch.device("cuda:0"))
    acc = gpu_lib.w4a8_gemm_i32(qx, tx, packed, N, workspace=ws)
    Y = gpu_lib.w4a8_gemm(qx, sx, tx, packed, s0, N, workspace=ws)
    rows = sample_rows(M)
    torch.cuda.synchronize()
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X[rows])
    assert np.array_equal(qx[rows].cpu().numpy(), qx_ref)
    acc_ref = oracle.gemm_i32(qx_ref, qhat)
    a = acc[rows].cpu().numpy()
    assert np.array_equal(a, acc_ref), f"{(a != acc_ref).sum()} sampled accumulators differ"
    check_y(Y[rows].cpu().numpy(), oracle.epilogue_f64(acc_ref, sx_ref, s0_ref))
    if ws.buf is not None:
        assert int(ws.buf.count_nonzero()) == 0


@pytest.mark.parametrize("name,N,K", PREFILL_SHAPES)
def test_prefill_per_channel_sampled_bit_exact(gpu_lib, name, N, K):
    """Per-channel W4A8 (NEXT-1) at M = 4096 on the planner's prefill tile."""
    M = 4096
    W = synth.weights_fp16(N, K, seed=N + K + 1)
    qu4_ref, sw_ref, zw_ref = oracle.pc_quantize(W)
    p_ref = oracle.pc_pack(qu4_ref)
    X, Xd = _acts(M, K)
    qx, sx, tx = gpu_lib.quantize_activations_per_token(Xd)
    acc = gpu_lib.pc_w4a8_gemm_i32(qx, tx, to_dev(p_ref), to_dev(zw_ref), N)
    rows = sample_rows(M)
    torch.cuda.synchronize()
    qx_ref, _, _ = oracle.quantize_activations(X[rows])
    acc_ref = oracle.pc_gemm_i32(qx_ref, qu4_ref, zw_ref)
    assert np.array_equal(acc[rows].cpu().numpy(), acc_ref)
