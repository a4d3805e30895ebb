"""GPU parity of the fused TP reduction (NEXT-3, qoq_w4a8_gemm_allreduce) through the C ABI.

One GPU is available here, so the cross-rank protocol is exercised without ranks that wait on one another:
  * world = 1: the push, the flag and the wait are local; Y must equal qoq_w4a8_gemm bit for bit, call after
    call (parities alternate, the call counter advances), also under CUDA-graph replay;
  * world = 2, 4, 8 with pre-seeded peers: every peer's partial, in the flag-in-data word format with this
    call's flag, is written into this rank's buffer BEFORE the single kernel runs (what the peers' kernels
    would have stored); this rank's kernel must store its own partial (with the flag) into every rank's slot
    and reduce in rank order exactly as oracle.tp_reduce_rank_order; as first, middle and last rank, 3 calls;
  * a peer whose words never arrive: the wait gives up after 2 s and sets the status word (no hang).
A real multi-GPU run (torchrun, NCCL + symmetric memory) is test_fused_reduction_multi_gpu, skipped with < 2 GPUs.
"""
import os
import subprocess
import sys

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


def _rank_inputs(M, N, K, seed):
    """One rank's row-parallel inputs: its K-shard weights and activations, quantized by the oracle."""
    W = synth.weights_fp16(N, K, seed=seed)
    X = synth.activations_fp16(M, K, seed=seed + 1)
    p, s0 = oracle.quantize_weights(W)
    qx, sx, tx = oracle.quantize_activations(X)
    return p, s0, qx, sx, tx


def _partial(M, N, K, case):
    """The rank's fp16 partial as the plain GEMM computes it (the fused kernel pushes exactly these bits)."""
    import paper_2405_04532_b200 as qoq
    p, s0, qx, sx, tx = case
    return qoq.w4a8_gemm(to_dev(qx), to_dev(sx), to_dev(tx), to_dev(p), to_dev(s0), N)


@pytest.mark.parametrize("M,N,K", [(64, 4096, 512), (1, 4096, 1792), (16, 1024, 256), (37, 512, 384),
                                   (130, 384, 256)])
def test_world1_equals_gemm_every_call(gpu_lib, M, N, K):
    case = _rank_inputs(M, N, K, seed=M + N + K)
    ref = _partial(M, N, K, case)
    p, s0, qx, sx, tx = (to_dev(a) for a in case)
    comm = gpu_lib.TpComm.local(M, N, dev())
    for call in range(5):   # parities 0, 1, 0, 1, 0; expected flag counts 1, 1, 2, 2, 3
        Y = gpu_lib.w4a8_gemm_allreduce(qx, sx, tx if call % 2 else None, p, s0, N, comm)
        torch.cuda.synchronize()
        assert torch.equal(Y, ref), f"call {call}"
    assert comm.status() == 0 and comm.calls() == 5
    y_ref = oracle.epilogue_f64(oracle.acc_from_packed(case[2], case[0], N, K), case[3], case[1])
    y = ref.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(y - y_ref) <= RTOL * np.abs(y_ref) + ATOL)


@pytest.mark.parametrize("M,N,K,mcap,ncap", [(37, 1280, 512, 64, 4096), (5, 256, 1792, 16, 512)])
def test_comm_larger_than_the_call(gpu_lib, M, N, K, mcap, ncap):
    """A comm sized for the largest call (m_cap > M, n_cap > N) serves smaller calls: the slots are pitched by
    the caps, at world 1 and with a pre-seeded peer at world 2."""
    cases = [_rank_inputs(M, N, K, seed=500 + r) for r in range(2)]
    parts = [_partial(M, N, K, c) for c in cases]
    comm1 = gpu_lib.TpComm.local(mcap, ncap, dev())
    p, s0, qx, sx, tx = (to_dev(a) for a in cases[0])
    for _ in range(2):
        assert torch.equal(gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm1), parts[0])
    recv = _rank_buffers(gpu_lib, mcap, ncap, 2)
    comm2 = gpu_lib.TpComm(0, 2, [r.data_ptr() for r in recv], mcap, ncap, dev(), keep=(recv,))
    want = torch.from_numpy(oracle.tp_reduce_rank_order([y.cpu().numpy() for y in parts])).to(dev())
    for call in range(2):
        par, flag = call & 1, call + 1
        _words(recv[0], par, 1, mcap, ncap)[:M, : N // 2].copy_(_ll(parts[1], flag))
        torch.cuda.synchronize()
        Y = gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm2)
        torch.cuda.synchronize()
        assert comm2.status() == 0 and torch.equal(Y, want)
        assert torch.equal(_words(recv[1], par, 0, mcap, ncap)[:M, : N // 2], _ll(parts[0], flag))
    assert comm1.status() == 0


def test_world1_cuda_graph_replay(gpu_lib):
    M, N, K = 64, 4096, 512
    case = _rank_inputs(M, N, K, seed=5)
    ref = _partial(M, N, K, case)
    p, s0, qx, sx, tx = (to_dev(a) for a in case)
    comm = gpu_lib.TpComm.local(M, N, dev())
    Y = torch.empty(M, N, dtype=torch.float16, device=dev())
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm, out=Y, stream=s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm, out=Y, stream=s)
    for _ in range(4):
        Y.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(Y, ref)
    assert comm.status() == 0 and comm.calls() == 1 + 3 * 4


def _rank_buffers(gpu_lib, M, N, world):
    return [torch.zeros(gpu_lib.tp_recv_bytes(world, M, N) // 4, dtype=torch.int32, device=dev()) for _ in range(world)]


def _words(buf, par, slot, M, N, world=2):
    """Slot `slot` of parity `par` of a receive buffer as [M][N/2] 8-byte words {2 fp16, flag}."""
    return buf.view(2, world, M, N // 2, 2)[par, slot]


def _ll(Y, flag):
    """An fp16 [M][N] partial in the flag-in-data word format (what a peer's kernel stores)."""
    M, N = Y.shape
    w = torch.empty(M, N // 2, 2, dtype=torch.int32, device=Y.device)
    w[..., 0] = Y.contiguous().view(torch.int32).view(M, N // 2)
    w[..., 1] = flag
    return w


@pytest.mark.parametrize("world,me", [(2, 0), (2, 1), (4, 2), (8, 0), (8, 7)])
@pytest.mark.parametrize("M,N,K", [(64, 4096, 512), (5, 512, 1792), (33, 1280, 256)])
def test_preseeded_peers_rank_order(gpu_lib, world, me, M, N, K):
    """One rank's kernel with world - 1 pre-seeded peers: every peer's partial (this call's flag) is in our buffer
    before the kernel runs; our partial must land in every peer's slot `me`, and Y must equal the rank-order
    reduction bit for bit."""
    cases = [_rank_inputs(M, N, K, seed=100 * (r + 1) + M) for r in range(world)]
    parts = [_partial(M, N, K, c) for c in cases]
    recv = _rank_buffers(gpu_lib, M, N, world)
    comm = gpu_lib.TpComm(me, world, [r.data_ptr() for r in recv], M, N, dev(), keep=(recv,))
    p, s0, qx, sx, tx = (to_dev(a) for a in cases[me])
    want = torch.from_numpy(oracle.tp_reduce_rank_order([y.cpu().numpy() for y in parts])).to(dev())
    for call in range(3):
        par, flag = call & 1, call + 1
        for q in range(world):   # what the peers' kernels store into OUR buffer (a stale flag would make us wait)
            if q != me:
                _words(recv[me], par, q, M, N, world).copy_(_ll(parts[q], flag))
        torch.cuda.synchronize()
        Y = gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm)
        torch.cuda.synchronize()
        assert comm.status() == 0
        assert torch.equal(Y, want), f"call {call}: rank-order reduction differs"
        for q in range(world):   # our partial, with this call's flag, in every rank's slot `me`
            assert torch.equal(_words(recv[q], par, me, M, N, world), _ll(parts[me], flag))
    # within the propagated north_star tolerance of the exact sum of the exact partials: each fp16 partial is
    # within RTOL |ref_q| + ATOL of its exact value, plus the final fp16 rounding
    refs = [oracle.epilogue_f64(oracle.acc_from_packed(c[2], c[0], N, K), c[3], c[1]) for c in cases]
    ref = sum(refs)
    y = Y.cpu().numpy().astype(np.float64)
    bound = sum(RTOL * np.abs(r) + ATOL for r in refs) + 2.0 ** -11 * np.abs(ref)
    assert np.all(np.abs(y - ref) <= bound)


def test_world2_stale_peer_times_out_without_hanging(gpu_lib):
    """The peer's slot holds the PREVIOUS call's words (flag 0 = never written): the reduction waits for this
    call's flag, gives up after 2 s and sets the status word instead of hanging."""
    M, N, K = 16, 256, 256
    mine = _rank_inputs(M, N, K, seed=9)
    recv = _rank_buffers(gpu_lib, M, N, 2)
    comm = gpu_lib.TpComm(0, 2, [r.data_ptr() for r in recv], M, N, dev(), keep=(recv,))
    p, s0, qx, sx, tx = (to_dev(a) for a in mine)
    gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm)
    torch.cuda.synchronize()
    assert comm.status() == 1


_MULTI = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["REPO"])
import paper_2405_04532_b200 as qoq, oracle, synth
from paper_2405_04532_b200 import parallel
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
M, N, K = 64, 4096, 512
comm = parallel.fused_tp_comm(qoq, dist.group.WORLD, M, N, dev)
parts, mine = [], None
for r in range(world):
    W = synth.weights_fp16(N, K, seed=300 + r); X = synth.activations_fp16(M, K, seed=400 + r)
    p, s0 = oracle.quantize_weights(W); qx, sx, tx = oracle.quantize_activations(X)
    t = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (qx, sx, tx, p, s0)]
    parts.append(qoq.w4a8_gemm(t[0], t[1], t[2], t[3], t[4], N).cpu().numpy())
    if r == rank: mine = t
want = oracle.tp_reduce_rank_order(parts)
for call in range(4):
    Y = qoq.w4a8_gemm_allreduce(mine[0], mine[1], mine[2], mine[3], mine[4], N, comm)
    torch.cuda.synchronize()
    assert comm.status() == 0, "peer wait timed out"
    assert np.array_equal(Y.cpu().numpy().view(np.uint16), want.view(np.uint16)), f"rank {rank} call {call}"
dist.barrier()
dist.destroy_process_group()
print("ok", rank)
'''


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs (the driver's multi-GPU runs)")
def test_fused_reduction_multi_gpu(tmp_path):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "tp_fused_multi.py"
    script.write_text(_MULTI)
    world = min(torch.cuda.device_count(), 8)
    env = dict(os.environ, REPO=root)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.count("ok") == world


@pytest.mark.parametrize("M", [1, 16, 64])
@pytest.mark.parametrize("N,K", [(8192, 1024), (8192, 3584), (8192, 3072), (4096, 512), (4096, 1792)])
def test_world1_row_parallel_shard_shapes(gpu_lib, M, N, K):
    """The row-parallel shard shapes of configs 4 / 5 (Llama-2-70B / Qwen1.5-72B at TP 8: o, down) and of
    Llama-3-8B at TP 8: the fused kernel (whole tiles, its own instantiation) equals the plain GEMM bit for bit."""
    case = _rank_inputs(M, N, K, seed=7 * M + K)
    ref = _partial(M, N, K, case)
    p, s0, qx, sx, tx = (to_dev(a) for a in case)
    comm = gpu_lib.TpComm.local(M, N, dev())
    Y = gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm)
    torch.cuda.synchronize()
    assert comm.status() == 0 and torch.equal(Y, ref)
