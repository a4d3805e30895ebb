"""GPU parity of the fused TP reduction (NEXT-3, qoq_w4a8_gemm_allreduce) through the C ABI.

One GPU is available here, so the cross-rank protocol is exercised without ranks that wait on one another:
  * world = 1: the push, the flag and the wait are local; Y must equal qoq_w4a8_gemm bit for bit, call after
    call (parities alternate, the call counter advances), also under CUDA-graph replay;
  * world = 2 with a pre-seeded peer: the peer's partial, in the flag-in-data word format with this call's
    flag, is written into this rank's buffer BEFORE the single kernel runs (what the peer's kernel would have
    stored); this rank's kernel must store its own partial (with the flag) into the peer's slot and reduce
    in rank order exactly as oracle.tp_reduce_rank_order; run as rank 0 and as rank 1, over 3 calls;
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


def _two_rank_buffers(gpu_lib, M, N):
    return [torch.zeros(gpu_lib.tp_recv_bytes(2, M, N) // 4, dtype=torch.int32, device=dev()) for _ in range(2)]


def _words(buf, par, slot, M, N):
    """Slot `slot` of parity `par` of a 2-rank receive buffer as [M][N/2] 8-byte words {2 fp16, flag}."""
    return buf.view(2, 2, M, N // 2, 2)[par, slot]


def _ll(Y, flag):
    """An fp16 [M][N] partial in the flag-in-data word format (what a peer's kernel stores)."""
    M, N = Y.shape
    w = torch.empty(M, N // 2, 2, dtype=torch.int32, device=Y.device)
    w[..., 0] = Y.contiguous().view(torch.int32).view(M, N // 2)
    w[..., 1] = flag
    return w


@pytest.mark.parametrize("me", [0, 1])
@pytest.mark.parametrize("M,N,K", [(64, 4096, 512), (5, 512, 1792), (33, 1280, 256)])
def test_world2_preseeded_peer_rank_order(gpu_lib, me, M, N, K):
    peer = 1 - me
    mine = _rank_inputs(M, N, K, seed=100 + M)
    theirs = _rank_inputs(M, N, K, seed=200 + M)
    Y_me = _partial(M, N, K, mine)
    Y_peer = _partial(M, N, K, theirs)
    recv = _two_rank_buffers(gpu_lib, M, N)
    comm = gpu_lib.TpComm(me, 2, [r.data_ptr() for r in recv], M, N, dev(), keep=(recv,))
    p, s0, qx, sx, tx = (to_dev(a) for a in mine)
    order = [None, None]
    order[me], order[peer] = Y_me.cpu().numpy(), Y_peer.cpu().numpy()
    want = torch.from_numpy(oracle.tp_reduce_rank_order(order)).to(dev())
    for call in range(3):
        par, flag = call & 1, call + 1
        # what the peer's kernel stores before our reduction can finish: its partial, with this call's flag,
        # in OUR slot `peer` (a stale flag would make us wait)
        _words(recv[me], par, peer, M, N).copy_(_ll(Y_peer, flag))
        torch.cuda.synchronize()
        Y = gpu_lib.w4a8_gemm_allreduce(qx, sx, tx, p, s0, N, comm)
        torch.cuda.synchronize()
        assert comm.status() == 0
        assert torch.equal(Y, want), f"call {call}: rank-order reduction differs"
        # our push landed in the peer's slot `me`: exactly the plain GEMM's partial, with this call's flag
        assert torch.equal(_words(recv[peer], par, me, M, N), _ll(Y_me, flag))
    # and the result is within the propagated north_star tolerance of the exact sum of the two exact partials:
    # each fp16 partial is within RTOL |ref_q| + ATOL of its exact value, plus the final fp16 rounding
    refs = [oracle.epilogue_f64(oracle.acc_from_packed(c[2], c[0], N, K), c[3], c[1]) for c in (mine, theirs)]
    ref = refs[0] + refs[1]
    y = Y.cpu().numpy().astype(np.float64)
    bound = sum(RTOL * np.abs(r) + ATOL for r in refs) + 2.0 ** -11 * np.abs(ref)
    assert np.all(np.abs(y - ref) <= bound)


def test_world2_stale_peer_times_out_without_hanging(gpu_lib):
    """The peer's slot holds the PREVIOUS call's words (flag 0 = never written): the reduction waits for this
    call's flag, gives up after 2 s and sets the status word instead of hanging."""
    M, N, K = 16, 256, 256
    mine = _rank_inputs(M, N, K, seed=9)
    recv = _two_rank_buffers(gpu_lib, M, N)
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
