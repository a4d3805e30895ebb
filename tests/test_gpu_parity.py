"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bit-exact: packed weights, s0, q_x, s_x, t_x and INT32 accumulators. FP16 Y within the north_star
tolerance |Y - y_ref| <= 2e-3 |y_ref| + 1e-3, y_ref the exact fp64 oracle value."""
import functools

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


def bits16(t):
    return t.cpu().numpy().view(np.uint16)


def check_y(Y, y_ref):
    y = Y.cpu().numpy().astype(np.float64)
    err = np.abs(y - y_ref)
    bad = err > RTOL * np.abs(y_ref) + ATOL
    assert not bad.any(), f"{bad.sum()} outputs outside tolerance; max err {err.max()}"


# ------------------------------------------------------------------ weights

@pytest.mark.parametrize("N,K", [(256, 256), (128, 128), (1280, 1024), (384, 4096)])
def test_quantize_weights_bit_exact(gpu_lib, N, K):
    W = synth.weights_fp16(N, K, seed=N + K)
    W[3] = 0                                   # zero row -> s0 = 1
    W[5] = np.float16(3e-7) * np.sign(W[5])    # underflowing row -> 2^-24 rule, clamp engaged
    W[7, :128] = np.abs(W[7, :128])            # an all-positive group (the Q4 corner)
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    p_ref, s0_ref = oracle.quantize_weights(W)
    assert np.array_equal(bits16(s0), s0_ref.view(np.uint16))
    assert np.array_equal(packed.cpu().numpy(), p_ref)


# ------------------------------------------------------------------ activations

@pytest.mark.parametrize("M,K,ldx", [(16, 256, 256), (1, 4096, 4096), (7, 128, 136), (65, 14336, 14336),
                                     (1000, 1024, 1024)])
def test_quantize_activations_bit_exact(gpu_lib, M, K, ldx):
    X = synth.activations_fp16(M, ldx, seed=M)
    if M > 3:
        X[2] = 0
        X[3] = np.float16(2e-6) * np.sign(X[3])   # s_x underflow / clamp regime
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X), K)
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X, K)
    assert np.array_equal(bits16(sx), sx_ref.view(np.uint16))
    assert np.array_equal(qx.cpu().numpy(), qx_ref)
    assert np.array_equal(tx.cpu().numpy(), tx_ref)


def test_quantize_activations_all_fp16_magnitudes(gpu_lib):
    """Every positive finite fp16 value as a row max (incl. subnormal-scale regimes)."""
    a = np.arange(1, 0x7c00, dtype=np.uint16).view(np.float16)
    X = np.zeros((a.size, 8), np.float16)
    X[:, 0] = a
    X[:, 1] = -a / 3
    X[:, 2] = a / 7
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    assert np.array_equal(bits16(sx), sx_ref.view(np.uint16))
    assert np.array_equal(qx.cpu().numpy(), qx_ref)


# ------------------------------------------------------------------ GEMM

def _case(M, N, K, seed):
    W = synth.weights_fp16(N, K, seed=seed)
    X = synth.activations_fp16(M, K, seed=seed)
    p_ref, s0_ref = oracle.quantize_weights(W)
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X)
    return W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref


GEMM_SHAPES = [(16, 256, 256), (1, 128, 128), (7, 256, 1024), (63, 1280, 256), (64, 128, 4096),
               (65, 384, 512), (129, 256, 384), (256, 512, 256), (300, 1280, 1024)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
@pytest.mark.parametrize("use_tx", [True, False])
def test_gemm_i32_bit_exact(gpu_lib, M, N, K, use_tx):
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=M * 7 + N + K)
    packed = to_dev(p_ref)
    acc = gpu_lib.w4a8_gemm_i32(to_dev(qx_ref), to_dev(tx_ref) if use_tx else None, packed, N)
    acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
    a = acc.cpu().numpy()
    assert np.array_equal(a, acc_ref), f"{(a != acc_ref).sum()} accumulators differ"


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_fp16_within_tolerance(gpu_lib, M, N, K):
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=M + 3 * N + K)
    Y = gpu_lib.w4a8_gemm(to_dev(qx_ref), to_dev(sx_ref), to_dev(tx_ref), to_dev(p_ref), to_dev(s0_ref), N)
    y_ref = oracle.epilogue_f64(oracle.acc_from_packed(qx_ref, p_ref, N, K), sx_ref, s0_ref)
    check_y(Y, y_ref)


def test_full_path_config1_and_workspace_restored(gpu_lib):
    """Config 1 end to end on device (quantize weights, quantize X, GEMM) and the split-K
    workspace returns to all-zero after the call."""
    M, N, K = 16, 256, 256
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=0)
    ws = gpu_lib.Workspace(dev())
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    Y = gpu_lib.w4a8_gemm(qx, sx, tx, packed, s0, N, workspace=ws)
    torch.cuda.synchronize()
    check_y(Y, oracle.linear_rows(X, p_ref, s0_ref, N))
    if ws.buf is not None:
        assert int(ws.buf.count_nonzero()) == 0
    # the one-call linear layer (fused quantization) on the same inputs: identical Y
    assert torch.equal(gpu_lib.linear(to_dev(X), packed, s0, N), Y)


def test_gemm_matches_library_w8a8_on_dequantized_weights(gpu_lib):
    """Library cross-check (W8A8 reduction, "as if it was W8A8"): the W4A8 accumulators equal
    cuBLASLt's INT8 GEMM (torch._int_mm) on the level-2-dequantized INT8 weights q̂."""
    M, N, K = 64, 1280, 1024
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=11)
    qu4, s, z = oracle.unpack(p_ref, N, K)
    qhat = oracle.dequant_level2(qu4, s, z).astype(np.int8)
    ref = torch._int_mm(to_dev(qx_ref), to_dev(qhat).t())   # [K][N] column-major view
    acc = gpu_lib.w4a8_gemm_i32(to_dev(qx_ref), to_dev(tx_ref), to_dev(p_ref), N)
    assert torch.equal(acc, ref)


@pytest.mark.parametrize("name,N,K", [(n, N, K) for n, N, K, _ in synth.LLAMA3_8B])
@pytest.mark.parametrize("M", [1, 64])
def test_llama3_8b_full_size_sampled(gpu_lib, name, N, K, M):
    """Full Llama-3-8B shapes at decode M in the launch configuration bench.py times: every output
    of sampled rows against the oracle (INT32 exact on the sample, Y within tolerance)."""
    W = synth.weights_fp16(N, K, seed=1)
    X = synth.activations_fp16(M, K, seed=1)
    p_ref, s0_ref = oracle.quantize_weights(W)
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    assert np.array_equal(packed.cpu().numpy(), p_ref)           # full-size packing, bit-exact
    assert np.array_equal(bits16(s0), s0_ref.view(np.uint16))
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    Y = gpu_lib.w4a8_gemm(qx, sx, tx, packed, s0, N)
    acc = gpu_lib.w4a8_gemm_i32(qx, tx, packed, N)
    rows = sorted({0, M - 1, M // 2})
    y_ref = oracle.linear_rows(X[rows], p_ref, s0_ref, N)
    check_y(Y[rows], y_ref)
    qx_ref, _, _ = oracle.quantize_activations(X[rows])
    acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
    assert np.array_equal(acc[rows].cpu().numpy(), acc_ref)


def test_linear_host_e2e(gpu_lib):
    M, N, K = 64, 1280, 1024
    W, X, p_ref, s0_ref, *_ = _case(M, N, K, seed=5)
    Xh = torch.from_numpy(X).pin_memory()
    Yh = torch.empty(M, N, dtype=torch.float16).pin_memory()
    scratch = torch.zeros(gpu_lib.linear_host_scratch_bytes(M, N, K), dtype=torch.uint8, device=dev())
    gpu_lib.linear_host(Xh, to_dev(p_ref), to_dev(s0_ref), N, Yh, scratch)
    torch.cuda.synchronize()
    check_y(Yh, oracle.linear_rows(X, p_ref, s0_ref, N))


@pytest.mark.parametrize("M", [1, 64])
def test_linear_host_shared_scratch_decode_shapes(gpu_lib, M):
    """The bench's e2e pattern: one scratch shared by the Llama-3-8B decode projections, called in a
    loop with H2D / D2H copies between launches. The sync words sit at offset 0 for every shape, so
    a larger shape's X copy never lands on a smaller shape's handshake counters (regression: the
    old [X][Y][workspace] layout moved the counters with K and faulted). Y must equal the two-call
    path (quantizer + GEMM) bit for bit on every pass."""
    shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
    gen = torch.Generator(device=dev()).manual_seed(5)
    packs, refs, hosts = [], [], []
    nbytes = max(gpu_lib.linear_host_scratch_bytes(M, N, K) for N, K in shapes)
    assert all(gpu_lib.gemm_workspace_bytes(M, N, K) == 0 for N, K in shapes)   # reuse rule holds
    scratch = torch.zeros(nbytes, dtype=torch.uint8, device=dev())
    for i, (N, K) in enumerate(shapes):
        W = (torch.randn(N, K, generator=gen, device=dev()) / K ** 0.5).half()
        p, s0 = gpu_lib.quantize_weights(W)
        X = torch.randn(M, K, generator=gen, device=dev()).half()
        qx, sx, tx = gpu_lib.quantize_activations_per_token(X)
        refs.append(gpu_lib.w4a8_gemm(qx, sx, tx, p, s0, N).cpu())
        packs.append((p, s0, N))
        hosts.append((X.cpu().pin_memory(), torch.empty(M, N, dtype=torch.float16).pin_memory()))
    for _ in range(3):
        for (p, s0, N), (Xh, Yh), ref in zip(packs, hosts, refs):
            Yh.zero_()
            gpu_lib.linear_host(Xh, p, s0, N, Yh, scratch)
            torch.cuda.synchronize()
            assert torch.equal(Yh, ref)
    assert int(scratch[:256].count_nonzero()) == 0


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("M,N,K", [(16, 256, 256), (1, 1280, 1024), (64, 512, 2048), (33, 384, 1152),
                                   (64, 4096, 4096)])
def test_gemm_all_planner_modes_bit_exact(gpu_lib, monkeypatch, mode, M, N, K):
    """Every work decomposition (0: whole tiles, 1: stream-K with the global workspace, 2: S-CTA
    cluster split-K reduced through DSMEM) gives the identical INT32 accumulators and Y."""
    monkeypatch.setenv("QOQ_FORCE_MODE", mode)
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=M + N + K + int(mode))
    ws = gpu_lib.Workspace(dev())
    acc = gpu_lib.w4a8_gemm_i32(to_dev(qx_ref), to_dev(tx_ref), to_dev(p_ref), N, workspace=ws)
    acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
    assert np.array_equal(acc.cpu().numpy(), acc_ref)
    Y = gpu_lib.w4a8_gemm(to_dev(qx_ref), to_dev(sx_ref), None, to_dev(p_ref), to_dev(s0_ref), N, workspace=ws)
    check_y(Y, oracle.epilogue_f64(acc_ref, sx_ref, s0_ref))
    torch.cuda.synchronize()
    if ws.buf is not None:
        assert int(ws.buf.count_nonzero()) == 0


def test_tp_shards_on_device(gpu_lib):
    """TP on the CUDA path (one GPU, shards run sequentially): column shards of the packed stream
    give bit-identical N-slices; row shards' INT32 accumulators (same q_x K-slices) sum exactly to
    the full accumulator."""
    from paper_2405_04532_b200 import parallel
    M, N, K, world = 16, 512, 1024, 4
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=21)
    packed, s0 = to_dev(p_ref), to_dev(s0_ref)
    qx, sx, tx = to_dev(qx_ref), to_dev(sx_ref), to_dev(tx_ref)
    full_acc = gpu_lib.w4a8_gemm_i32(qx, tx, packed, N)
    full_y = gpu_lib.w4a8_gemm(qx, sx, tx, packed, s0, N)
    cols = []
    for r in range(world):
        p_r, s0_r = parallel.shard_packed(packed, s0, N, K, "col", r, world)
        cols.append(gpu_lib.w4a8_gemm(qx, sx, tx, p_r.contiguous(), s0_r.contiguous(), N // world))
    assert torch.equal(torch.cat(cols, dim=1), full_y)
    tot = torch.zeros_like(full_acc)
    for r in range(world):
        p_r, _ = parallel.shard_packed(packed, s0, N, K, "row", r, world)
        qx_r = parallel.shard_input(qx, "row", r, world).contiguous()
        tot += gpu_lib.w4a8_gemm_i32(qx_r, None, p_r.contiguous(), N)
    assert torch.equal(tot, full_acc)


@pytest.mark.parametrize("mode", ["0", "1", "2"])
@pytest.mark.parametrize("M,N,K", [
    (16, 19200, 640),    # BN=16: 150 tiles > 148 SMs (persistent CTAs own 2 tiles), KS=3 (odd)
    (5, 2560, 1408),     # BN=16: KT=11 -> last step holds one k-tile; odd-length stream-K segments
    (40, 1280, 3200),    # BN=64: KS=13
    (64, 19200, 384),    # BN=64: 150 tiles, KS=2 with a 1-tile last step
    (100, 1280, 1664),   # BN=128: KS=7
    (200, 768, 2688),    # M > 128: the planner's prefill tile (BN = 128 here: 6 tiles < #SMs), KS=11
])
def test_gemm_segment_edge_cases_bit_exact(gpu_lib, monkeypatch, mode, M, N, K):
    """Odd step counts, 1-tile last steps, multi-tile persistent CTAs and odd-length split-K
    segments in every decomposition: the pipeline rings and the two MMA issuers' accumulators must
    still give the exact INT32 sums."""
    monkeypatch.setenv("QOQ_FORCE_MODE", mode)
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=M + K)
    for use_tx in (True, False):
        acc = gpu_lib.w4a8_gemm_i32(to_dev(qx_ref), to_dev(tx_ref) if use_tx else None, to_dev(p_ref), N)
        acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
        a = acc.cpu().numpy()
        assert np.array_equal(a, acc_ref), f"{(a != acc_ref).sum()} accumulators differ (tx={use_tx})"


@pytest.mark.parametrize("mode", ["0", "1"])
@pytest.mark.parametrize("M,N,K", [(64, 256, 256), (33, 1280, 1024), (64, 4096, 4096), (100, 512, 1664),
                                   (256, 1024, 384), (40, 2560, 3200)])
def test_gemm_cta_pair_bit_exact(gpu_lib, monkeypatch, mode, M, N, K):
    """CTA-pair (cluster of 2, tcgen05 cta_group::2, M = 256) variant of the GEMM: the pair's
    accumulators equal the oracle's exactly in both decompositions it supports."""
    monkeypatch.setenv("QOQ_FORCE_MODE", mode)
    monkeypatch.setenv("QOQ_FORCE_CG", "2")
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=M * 3 + K)
    ws = gpu_lib.Workspace(dev())
    for use_tx in (True, False):
        acc = gpu_lib.w4a8_gemm_i32(to_dev(qx_ref), to_dev(tx_ref) if use_tx else None, to_dev(p_ref), N,
                                    workspace=ws)
        assert np.array_equal(acc.cpu().numpy(), oracle.acc_from_packed(qx_ref, p_ref, N, K))
    Y = gpu_lib.w4a8_gemm(to_dev(qx_ref), to_dev(sx_ref), to_dev(tx_ref), to_dev(p_ref), to_dev(s0_ref), N,
                          workspace=ws)
    check_y(Y, oracle.epilogue_f64(oracle.acc_from_packed(qx_ref, p_ref, N, K), sx_ref, s0_ref))


# ------------------------------------------------------------------ fused linear (quantize + GEMM)

FUSED_SHAPES = [
    (1, 128, 128, 128),       # one tile, one CTA quantizes the only row
    (16, 256, 256, 264),      # ldx > K (a TP K-shard view)
    (33, 1280, 1024, 1024),
    (64, 4096, 4096, 4096),   # decode o_proj
    (64, 128, 4096, 4096),    # one output tile: few CTAs, each quantizes many rows
    (64, 19200, 384, 384),    # 150 tiles > 148 SMs: persistent CTAs, every SM in the handshake
    (5, 2560, 1408, 1408),
    (48, 1024, 14336, 14336), # long rows (down_proj K)
    (65, 512, 1024, 1024),    # above the fusion limit: quantizer kernel + GEMM
    (300, 1280, 1024, 1024),
]


def _fused_case(M, N, K, ldx, seed):
    W = synth.weights_fp16(N, K, seed=seed)
    X = synth.activations_fp16(M, ldx, seed=seed)
    if M > 3:
        X[2] = 0
        X[3] = np.float16(2e-6) * np.sign(X[3])
    p_ref, s0_ref = oracle.quantize_weights(W)
    qx_ref, sx_ref, tx_ref = oracle.quantize_activations(X, K)
    return X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref


# the two-kernel path is covered by the GEMM parity tests; auto / 2 suffice for it here
PATH_MODES = [("fused", m) for m in ("auto", "0", "1", "2", "cg2")] + [("two", "auto"), ("two", "2")]


@pytest.mark.parametrize("path,mode", PATH_MODES)
@pytest.mark.parametrize("M,N,K,ldx", FUSED_SHAPES)
def test_fused_linear_bit_exact(gpu_lib, monkeypatch, path, mode, M, N, K, ldx):
    """qoq_w4a8_linear, on the fused path (QOQ_LINEAR_FUSED=1: per-token quantization inside the
    GEMM for M <= 64) and on the default quantizer + GEMM chain: the quantized activations it leaves
    in the workspace equal the oracle's bit for bit, Y is bit-identical to the two-call path
    (quantizer + GEMM) and within tolerance of the oracle, and repeated launches on the same
    workspace (grid-handshake counters re-zeroed by the last CTA) stay exact."""
    if path == "fused":
        monkeypatch.setenv("QOQ_LINEAR_FUSED", "1")
    else:
        monkeypatch.delenv("QOQ_LINEAR_FUSED", raising=False)
    if mode == "cg2":
        monkeypatch.setenv("QOQ_FORCE_CG", "2")
    elif mode != "auto":
        monkeypatch.setenv("QOQ_FORCE_MODE", mode)
    X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _fused_case(M, N, K, ldx, seed=M + N + K)
    Xd, packed, s0 = to_dev(X), to_dev(p_ref), to_dev(s0_ref)
    nbytes = gpu_lib.linear_workspace_bytes(M, N, K)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev())

    class _WS:   # caller-owned workspace (exact size) so its contents can be inspected
        def get(self, n):
            return ws, ws.numel()

    two = gpu_lib.w4a8_gemm(to_dev(qx_ref), to_dev(sx_ref), to_dev(tx_ref), packed, s0, N)
    y_ref = oracle.epilogue_f64(oracle.acc_from_packed(qx_ref, p_ref, N, K), sx_ref, s0_ref)
    for rep in range(3):
        Y = gpu_lib.w4a8_linear(Xd, packed, s0, N, K, workspace=_WS())
        torch.cuda.synchronize()
        assert torch.equal(Y, two), f"rep {rep}: fused Y differs from quantizer + GEMM"
        check_y(Y, y_ref)
        qx, sx, tx = gpu_lib.linear_workspace_views(ws, M, N, K)
        assert np.array_equal(qx.cpu().numpy(), qx_ref)
        assert np.array_equal(bits16(sx), sx_ref.view(np.uint16))
        assert np.array_equal(tx.cpu().numpy(), tx_ref)
        assert int(ws[:256].count_nonzero()) == 0, "handshake counters not re-zeroed"
        o = 256 + (gpu_lib.gemm_workspace_bytes(M, N, K) + 255) // 256 * 256
        assert int(ws[256:o].count_nonzero()) == 0, "split-K workspace not restored"


@pytest.mark.parametrize("path", ["fused", "two"])
def test_fused_linear_in_cuda_graph(gpu_lib, monkeypatch, path):
    """w4a8_linear (fused kernel, or quantizer + GEMM) replayed from a CUDA graph (frozen arguments,
    same workspace every replay) with changing activations: every replay quantizes the new X and
    matches the oracle."""
    if path == "fused":
        monkeypatch.setenv("QOQ_LINEAR_FUSED", "1")
    else:
        monkeypatch.delenv("QOQ_LINEAR_FUSED", raising=False)
    M, N, K = 64, 1280, 1024
    X0, p_ref, s0_ref, *_ = _fused_case(M, N, K, K, seed=77)
    packed, s0 = to_dev(p_ref), to_dev(s0_ref)
    Xd = to_dev(X0)
    ws = gpu_lib.Workspace(dev())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        Y = gpu_lib.w4a8_linear(Xd, packed, s0, N, workspace=ws, stream=s)
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gpu_lib.w4a8_linear(Xd, packed, s0, N, out=Y, workspace=ws, stream=s)
    for seed in (1, 2, 3):
        X = synth.activations_fp16(M, K, seed=seed)
        Xd.copy_(to_dev(X))
        g.replay()
        torch.cuda.synchronize()
        check_y(Y, oracle.linear_rows(X, p_ref, s0_ref, N))


def test_default_workspace_per_launch_stream(gpu_lib, monkeypatch):
    """the default workspace is keyed by the stream the call LAUNCHES on (not torch's
    current stream). Stream-K GEMMs (mode 1: split-K partials and tile counters in the workspace,
    zero on entry) issued back to back on two explicit streams, with no ordering between them, must
    each give the exact accumulators."""
    monkeypatch.setenv("QOQ_FORCE_MODE", "1")
    M, N, K = 64, 1280, 3200
    W, X, p_ref, s0_ref, qx_ref, sx_ref, tx_ref = _case(M, N, K, seed=91)
    acc_ref = oracle.acc_from_packed(qx_ref, p_ref, N, K)
    qx, tx, packed = to_dev(qx_ref), to_dev(tx_ref), to_dev(p_ref)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(8):
        outs.append(gpu_lib.w4a8_gemm_i32(qx, tx, packed, N, stream=s1))
        outs.append(gpu_lib.w4a8_gemm_i32(qx, tx, packed, N, stream=s2))
    torch.cuda.synchronize()
    for a in outs:
        assert np.array_equal(a.cpu().numpy(), acc_ref)


def _tp_shard_cases():
    """BASELINE configs 4 and 5: the per-rank GEMM shapes of Llama-2-70B at TP 2 / 4 / 8 and Qwen1.5-72B at
    TP 8 (column-parallel N / TP, row-parallel K / TP; gate and up fused), the shapes each rank's kernel runs."""
    from paper_2405_04532_b200 import parallel
    cases = []
    for model, tps in (("llama2-70b", (2, 4, 8)), ("qwen1.5-72b", (8,))):
        for tp in tps:
            for name, Nr, Kr, N, K, kind, qg in parallel.rank_layer_plan(synth.fuse_gate_up(synth.MODELS[model][0]), tp):
                cases.append((f"{model}-tp{tp}-{name}", Nr, Kr))
    return cases


@functools.lru_cache(maxsize=2)
def _shard_weights(N, K):
    W = synth.weights_fp16(N, K, seed=3)
    p_ref, s0_ref = oracle.quantize_weights(W)
    return W, p_ref, s0_ref


@pytest.mark.parametrize("M", [1, 64, 1024])
@pytest.mark.parametrize("case,N,K", _tp_shard_cases())
def test_tp_shard_shapes_sampled(gpu_lib, case, N, K, M):
    """Every rank-shard GEMM of configs 4 / 5 at decode and prefill M, in the planner's launch configuration:
    INT32 exact and Y within tolerance on sampled token rows (first, middle, last)."""
    W, p_ref, s0_ref = _shard_weights(N, K)
    X = synth.activations_fp16(M, K, seed=3)
    packed, s0 = gpu_lib.quantize_weights(to_dev(W))
    assert np.array_equal(packed.cpu().numpy(), p_ref)
    qx, sx, tx = gpu_lib.quantize_activations_per_token(to_dev(X))
    Y = gpu_lib.w4a8_gemm(qx, sx, tx, packed, s0, N)
    acc = gpu_lib.w4a8_gemm_i32(qx, tx, packed, N)
    rows = sorted({0, M - 1, M // 2})
    check_y(Y[rows], oracle.linear_rows(X[rows], p_ref, s0_ref, N))
    qx_ref, _, _ = oracle.quantize_activations(X[rows])
    assert np.array_equal(acc[rows].cpu().numpy(), oracle.acc_from_packed(qx_ref, p_ref, N, K))
