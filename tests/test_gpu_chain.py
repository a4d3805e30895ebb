"""GPU parity of the persistent decode chain (qoq_w4a8_linear_chain, ABI v6): n linear layers in ONE
launch must give, for every linear, Y bit-identical to the per-call path (qoq_w4a8_linear = the
per-token quantizer + the W4A8 GEMM, itself bit-exact in INT32 against the oracle) and within the
north_star tolerance of the oracle (|Y - y_ref| <= 2e-3 |y_ref| + 1e-3, y_ref exact fp64), including
chains where a linear's input IS an earlier linear's output (the grid-wide dependency), odd k-tile
counts, more output tiles than SMs, M from 1 to 128, row-strided inputs, repeated launches on one
workspace and CUDA-graph replay."""
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


def check_y(y, y_ref):
    y = np.asarray(y, np.float64)
    err = np.abs(y - y_ref)
    bad = err > RTOL * np.abs(y_ref) + ATOL
    assert not bad.any(), f"{bad.sum()} outputs outside tolerance; max err {err.max()}"


def make_layers(M, shapes, seed, chained=False, ldx_pad=0):
    """shapes [(N, K)]; chained: X_{j+1} = Y_j (needs N_j == K_{j+1}). Returns (layers, host refs)."""
    layers, host = [], []
    prevY = None
    for j, (N, K) in enumerate(shapes):
        W = synth.weights_fp16(N, K, seed=seed + 31 * j)
        p_ref, s0_ref = oracle.quantize_weights(W)
        if chained and prevY is not None:
            X = prevY
        else:
            Xh = synth.activations_fp16(M, K + ldx_pad, seed=seed + 7 * j)
            X = to_dev(Xh)
        Y = torch.full((M, N), float("nan"), dtype=torch.float16, device=dev())
        layers.append((X, to_dev(p_ref), to_dev(s0_ref), N, Y, K))
        host.append((p_ref, s0_ref))
        prevY = Y
    return layers, host


def sequential(gpu_lib, layers):
    """The per-call path on fresh outputs, in order (chained inputs follow the chain's own Ys)."""
    outs = []
    remap = {}
    for X, packed, s0, N, Y, K in layers:
        Xs = remap.get(X.data_ptr(), X)
        out = gpu_lib.w4a8_linear(Xs, packed, s0, N, K)
        remap[Y.data_ptr()] = out
        outs.append(out)
    return outs


SHAPE_SETS = {
    "small": [(256, 256), (1280, 1024), (384, 1152), (128, 128)],
    "wide": [(19200, 384), (256, 2304)],                         # 150 tiles > 148 SMs; KT = 18
    "long_k": [(512, 14336), (4096, 512)],                        # K = 14336 (two-pass quantizer)
}


@pytest.mark.parametrize("M", [1, 5, 16, 33, 64, 100, 128])
@pytest.mark.parametrize("shapes", ["small", "wide", "long_k"])
def test_chain_matches_per_call_path_and_oracle(gpu_lib, M, shapes):
    layers, host = make_layers(M, SHAPE_SETS[shapes], seed=M * 3 + len(shapes))
    ref = sequential(gpu_lib, layers)
    gpu_lib.w4a8_linear_chain(layers)
    torch.cuda.synchronize()
    for j, ((X, packed, s0, N, Y, K), r, (p_ref, s0_ref)) in enumerate(zip(layers, ref, host)):
        assert torch.equal(Y, r), f"linear {j}: chain Y differs from the per-call path"
        rows = sorted({0, M // 2, M - 1})
        check_y(Y[rows].cpu().numpy(), oracle.linear_rows(X[rows].cpu().numpy(), p_ref, s0_ref, N, K=K))


@pytest.mark.parametrize("M", [1, 16, 64])
def test_chain_dependent_inputs(gpu_lib, M):
    """X_{j+1} = Y_j: each quantization must see the complete previous output (grid-wide ordering)."""
    shapes = [(1024, 512), (2048, 1024), (512, 2048), (1280, 512), (512, 1280)]
    layers, host = make_layers(M, shapes, seed=40 + M, chained=True)
    ref = sequential(gpu_lib, layers)
    gpu_lib.w4a8_linear_chain(layers)
    torch.cuda.synchronize()
    Xcur = layers[0][0].cpu().numpy()
    for j, ((X, packed, s0, N, Y, K), r, (p_ref, s0_ref)) in enumerate(zip(layers, ref, host)):
        assert torch.equal(Y, r), f"linear {j}"
        check_y(Y.cpu().numpy(), oracle.linear_rows(Xcur, p_ref, s0_ref, N))
        Xcur = Y.cpu().numpy()


def test_chain_strided_inputs_and_workspace_reuse(gpu_lib):
    """ldx > K (a K-view of wider rows), and one workspace reused by chains of different shapes and
    M (the default workspace of the other tests is shared the same way): every call leaves the
    counter head zero for the next, and nothing else needs initializing."""
    ws = gpu_lib.Workspace(dev())
    for M, shapes, pad in ((64, SHAPE_SETS["small"], 64), (7, SHAPE_SETS["wide"], 0), (64, SHAPE_SETS["long_k"], 8)):
        layers, host = make_layers(M, shapes, seed=M + pad, ldx_pad=pad)
        ref = sequential(gpu_lib, layers)
        for rep in range(3):
            gpu_lib.w4a8_linear_chain(layers, workspace=ws)
            torch.cuda.synchronize()
            for (X, packed, s0, N, Y, K), r in zip(layers, ref):
                assert torch.equal(Y, r), f"M={M} rep {rep}"
        # the zero-required head (grid and tile counters, 12288 bytes) is zero again after every call
        assert int(ws.buf[:12288].count_nonzero()) == 0


def test_chain_llama3_8b_decode_layers_in_graph(gpu_lib):
    """Two Llama-3-8B decode layers (qkv, o, gate_up, down) at M = 64 as one chain, captured in a CUDA
    graph and replayed with new activations: bit-identical to the per-call path every replay, and
    sampled rows within tolerance of the oracle."""
    M = 64
    shapes = [(N, K) for _, N, K, _ in synth.fuse_gate_up(synth.LLAMA3_8B)] * 2
    gen = torch.Generator(device=dev()).manual_seed(5)
    layers = []
    for j, (N, K) in enumerate(shapes):
        W = (torch.randn(N, K, generator=gen, device=dev()) / K ** 0.5).half()
        p, s0 = gpu_lib.quantize_weights(W)
        X = synth.device_activations_fp16(M, K, gen, dev())
        layers.append((X, p, s0, N, torch.empty(M, N, dtype=torch.float16, device=dev()), K))
    ws = gpu_lib.Workspace(dev())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gpu_lib.w4a8_linear_chain(layers, workspace=ws, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gpu_lib.w4a8_linear_chain(layers, workspace=ws, stream=s)
    for rep in range(3):
        for X, *_ in layers:
            X.copy_(synth.device_activations_fp16(M, X.shape[1], gen, dev()))
        g.replay()
        torch.cuda.synchronize()
        ref = sequential(gpu_lib, layers)
        for j, ((X, p, s0, N, Y, K), r) in enumerate(zip(layers, ref)):
            assert torch.equal(Y, r), f"rep {rep} linear {j}"
    X, p, s0, N, Y, K = layers[3]                                     # down_proj, sampled vs the oracle
    rows = [0, 31, 63]
    p_ref = p.cpu().numpy()
    check_y(Y[rows].cpu().numpy(), oracle.linear_rows(X[rows].cpu().numpy(), p_ref, s0.cpu().numpy(), N))
