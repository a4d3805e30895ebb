"""GPU parity for the per-channel W4A8 path (NEXT-1, §5.2.2) through the C ABI against the
CPU oracle: packed codes, s_w and z_w bit-exact; INT32 Σ q_x (q_u4 − z_w) bit-exact in every
planner mode; FP16 Y within the north_star tolerance of the exact fp64 value."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-3, 1e-3


def dev():
    return torch.device("cuda:0")


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev())


def check_y(Y, y_ref):
    y = Y.cpu().numpy().astype(np.float64)
    err = np.abs(y - y_ref)
    bad = err > RTOL * np.abs(y_ref) + ATOL
    assert not bad.any(), f"{bad.sum()} outputs outside tolerance; max err {err.max()}"


def special_weights(N, K, seed):
    W = synth.weights_fp16(N, K, seed=seed)
    W[1] = 0                                                       # range 0 -> s_w = 1, z = 0
    W[2] = np.float16(0.25)                                        # constant row
    W[3] = np.abs(W[3])                                            # all-positive: z clamps to 0
    W[4] = -np.abs(W[4])                                           # all-negative: z clamps to 15
    W[5] = np.float16(3e-7) * np.sign(W[5])                        # s_w underflow -> 2^-24
    q = np.random.default_rng(seed).integers(0, 16, K)
    q[:2] = (0, 15)
    W[6] = ((q - 7) * 2.0 ** -6).astype(np.float16)                # an exact grid (ties at t + z)
    W[7, :6] = (np.array([0, 15, 4.5, 0.5, 1.5, 7.5]) * 2.0 ** -4).astype(np.float16)
    W[7, 6:] = 0
    return W


@pytest.mark.parametrize("N,K", [(256, 256), (128, 128), (1280, 1024), (384, 4096)])
def test_pc_quantize_weights_bit_exact(gpu_lib, N, K):
    W = special_weights(N, K, seed=N + K)
    packed, s_w, z_w = gpu_lib.pc_quantize_weights(to_dev(W))
    p_ref, s_ref, z_ref = oracle.pc_quantize_weights(W)
    assert np.array_equal(s_w.cpu().numpy().view(np.uint16), s_ref.view(np.uint16))
    assert np.array_equal(z_w.cpu().numpy(), z_ref)
    assert np.array_equal(packed.cpu().numpy(), p_ref)


PC_SHAPES = [(16, 256, 256), (1, 1280, 1024), (64, 512, 2048), (33, 384, 1152), (64, 4096, 4096),
             (130, 1024, 1024), (300, 1280, 512), (5, 256, 14336)]


@pytest.mark.parametrize("mode", ["auto", "0", "1", "2"])
@pytest.mark.parametrize("M,N,K", PC_SHAPES)
def test_pc_gemm_i32_and_fp16_bit_exact(gpu_lib, monkeypatch, mode, M, N, K):
    if mode != "auto":
        monkeypatch.setenv("QOQ_FORCE_MODE", mode)
    W = special_weights(N, K, seed=M + N + K)
    X = synth.activations_fp16(M, K, seed=M + K)
    if M > 3:
        X[2] = 0
    p_ref, s_ref, z_ref = oracle.pc_quantize_weights(W)
    qx, sx, tx = oracle.quantize_activations(X)
    acc_ref = oracle.pc_acc_from_packed(qx, p_ref, z_ref, N, K)
    packed, s_w, z_w, qxd, sxd, txd = map(to_dev, (p_ref, s_ref, z_ref, qx, sx, tx))
    acc = gpu_lib.pc_w4a8_gemm_i32(qxd, txd, packed, z_w, N)
    assert np.array_equal(acc.cpu().numpy(), acc_ref)
    Y = gpu_lib.pc_w4a8_gemm(qxd, sxd, txd, packed, s_w, z_w, N)
    check_y(Y, oracle.epilogue_f64(acc_ref, sx, s_ref))


@pytest.mark.parametrize("N,K", [(4096, 14336), (28672, 4096)])
def test_pc_full_size_sampled_rows(gpu_lib, N, K):
    """Llama-3-8B down / fused gate_up at decode M = 64, the bench's launch configuration: the GPU
    packer's output feeds the GEMM; sampled rows are checked against the oracle one by one."""
    M = 64
    W = synth.weights_fp16(N, K, seed=7)
    X = synth.activations_fp16(M, K, seed=7)
    packed, s_w, z_w = gpu_lib.pc_quantize_weights(to_dev(W))
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    Y = gpu_lib.pc_w4a8_gemm(qx, sx, tx, packed, s_w, z_w, N).cpu().numpy().astype(np.float64)
    rows = np.random.default_rng(0).choice(N, 96, replace=False)
    qu4, s_ref, z_ref = oracle.pc_quantize(W[rows])
    assert np.array_equal(s_w.cpu().numpy()[rows].view(np.uint16), s_ref.view(np.uint16))
    assert np.array_equal(z_w.cpu().numpy()[rows], z_ref)
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    y_ref = oracle.epilogue_f64(oracle.pc_gemm_i32(qx_ref, qu4, z_ref), sx_ref, s_ref)
    err = np.abs(Y[:, rows] - y_ref)
    assert not (err > RTOL * np.abs(y_ref) + ATOL).any(), err.max()
