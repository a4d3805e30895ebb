"""Tensor-parallel host logic on CPU: world_size 2 over `gloo` (reading Q17).

Per-rank math is the CPU oracle (the per-rank GEMM itself is parity-tested on the GPU); what is
checked here is the sharding and the reduction:
  * column-parallel: each rank's slice is bit-identical to the 1-GPU oracle result on that slice;
  * row-parallel: the all-reduced fp16 partials match the fp64 sum of the per-rank exact results
    within the north_star tolerance, and approximate the 1-GPU result.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2405_04532_b200 import parallel

RTOL, ATOL = 2e-3, 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_linear(X_r, shard):
    """Rank-local W4A8 linear on the CPU oracle from a packed shard: quantize X_r per token, GEMM, fp16."""
    packed, s0, N = shard
    X = np.ascontiguousarray(X_r)
    y = oracle.linear_rows(X, np.ascontiguousarray(packed), np.ascontiguousarray(s0), N)
    return torch.from_numpy(y.astype(np.float16))


def _packed_shard(W, kind, rank, world):
    """Quantize the full weight once (oracle packer), then shard the packed stream."""
    N, K = W.shape
    packed, s0 = oracle.quantize_weights(W)
    p_r, s0_r = parallel.shard_packed(packed, s0, N, K, kind, rank, world)
    return p_r, s0_r, (N // world if kind == "col" else N)


def _worker(rank, world, port, kind, M, N, K, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # TP weights scaled 1/4 (SURVEY §8(d) "Row-parallel TP parity: W ~ N(0, 1/(16K))")
        W = synth.weights_fp16(N, K, seed=3, std_scale=0.25)
        X = synth.activations_fp16(M, K, seed=3)
        W_r = _packed_shard(W, kind, rank, world)

        def all_reduce(Y):
            dist.all_reduce(Y, op=dist.ReduceOp.SUM)

        Y = parallel.tp_linear(X, W_r, kind, _oracle_linear, all_reduce, rank, world)
        out_q.put((rank, Y.numpy()))
    finally:
        dist.destroy_process_group()


def _run(kind, M, N, K, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, M, N, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_shard_helpers():
    W = np.arange(256 * 512).reshape(256, 512)
    assert parallel.shard_weight(W, "col", 1, 2).shape == (128, 512)
    assert parallel.shard_weight(W, "row", 1, 2).shape == (256, 256)
    assert np.array_equal(parallel.shard_weight(W, "row", 1, 2), W[:, 256:])
    with pytest.raises(ValueError):
        parallel.shard_weight(W, "col", 0, 4)       # 256 / 4 = 64 is not a multiple of 128
    with pytest.raises(ValueError):
        parallel.check_shardable(1280, 8192, "row", 3)
    # every Llama-2-70B / Qwen1.5-72B TP shard of BASELINE configs 3-4 is group-aligned
    for model in ("llama2-70b", "qwen1.5-72b"):
        for _, N, K, kind in synth.MODELS[model][0]:
            for tp in (2, 4, 8):
                parallel.check_shardable(N, K, kind, tp)


def test_column_parallel_gloo_bit_identical_slices():
    M, N, K = 8, 256, 256
    res = _run("col", M, N, K)
    W = synth.weights_fp16(N, K, seed=3, std_scale=0.25)
    X = synth.activations_fp16(M, K, seed=3)
    packed, s0 = oracle.quantize_weights(W)
    full = _oracle_linear(X, (packed, s0, N)).numpy()
    got = np.concatenate([res[0], res[1]], axis=1)
    assert np.array_equal(got.view(np.uint16), full.view(np.uint16))


def test_row_parallel_gloo_allreduce_within_tolerance():
    M, N, K = 8, 128, 512
    res = _run("row", M, N, K)
    assert np.array_equal(res[0].view(np.uint16), res[1].view(np.uint16))   # all ranks agree
    W = synth.weights_fp16(N, K, seed=3, std_scale=0.25)
    X = synth.activations_fp16(M, K, seed=3)
    ref = np.zeros((M, N))
    for r in range(2):
        p_r, s0_r, _ = _packed_shard(W, "row", r, 2)
        Xr = parallel.shard_input(X, "row", r, 2)
        ref += oracle.linear_rows(np.ascontiguousarray(Xr), p_r, s0_r, N)
    y = res[0].astype(np.float64)
    assert np.all(np.abs(y - ref) <= RTOL * np.abs(ref) + ATOL)
    # Same quantized weights as 1 GPU; only the per-token activation scales are per-rank (Q17), so
    # the TP result stays close to the 1-GPU layer and inside the float layer's envelope.
    fl = X.astype(np.float64) @ W.astype(np.float64).T
    packed, s0 = oracle.quantize_weights(W)
    one = oracle.linear_rows(X, packed, s0, N)
    assert np.linalg.norm(y - one) / np.linalg.norm(one) < 0.05
    assert np.linalg.norm(y - fl) / np.linalg.norm(fl) < 0.2


def test_packed_row_shards_sum_to_the_full_accumulator():
    """With the per-rank activation quantization replaced by the 1-GPU q_x (a K-slice of it), the
    INT32 partials of the row shards sum EXACTLY to the 1-GPU accumulators: the shard operation on
    the tile stream loses nothing."""
    M, N, K = 4, 256, 768
    W = synth.weights_fp16(N, K, seed=5)
    X = synth.activations_fp16(M, K, seed=5)
    packed, s0 = oracle.quantize_weights(W)
    qx, _, _ = oracle.quantize_activations(X)
    full = oracle.acc_from_packed(qx, packed, N, K)
    tot = np.zeros_like(full)
    for r in range(3):
        p_r, _ = parallel.shard_packed(packed, s0, N, K, "row", r, 3)
        qx_r = np.ascontiguousarray(parallel.shard_input(qx, "row", r, 3))
        tot += oracle.acc_from_packed(qx_r, p_r, N, K // 3)
    assert np.array_equal(tot, full)


# ---- TP FFN with the SiLU·mul quantization fused (NEXT-2) over gloo ----

def _mlp_weights(I, K):
    Wg = synth.weights_fp16(I, K, seed=7, std_scale=0.25)
    Wu = synth.weights_fp16(I, K, seed=8, std_scale=0.25)
    Wd = synth.weights_fp16(K, I, seed=9, std_scale=0.25)
    return Wg, Wu, Wd


def _mlp_oracle_act_linear(GU_r, shard):
    """silu_mul_quantize of [gate_r | up_r] (oracle, Q23) + the W4A8 GEMM of the down shard."""
    packed, s0, N = shard
    GU = GU_r.numpy() if hasattr(GU_r, "numpy") else GU_r
    qx, sx, tx = oracle.silu_mul_quantize(np.ascontiguousarray(GU))
    acc = oracle.acc_from_packed(qx, np.ascontiguousarray(packed), N, qx.shape[1])
    y = oracle.epilogue_f64(acc, sx, np.ascontiguousarray(s0))
    return torch.from_numpy(y.astype(np.float16))


def _mlp_worker(rank, world, port, M, I, K, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Wg, Wu, Wd = _mlp_weights(I, K)
        X = synth.activations_fp16(M, K, seed=7)
        a, b = parallel.gate_up_shard_rows(I, rank, world)
        gu = np.ascontiguousarray(np.concatenate([Wg[a:b], Wu[a:b]], axis=0))
        p_gu, s_gu = oracle.quantize_weights(gu)
        p_d, s_d = oracle.quantize_weights(Wd)
        p_dr, s_dr = parallel.shard_packed(p_d, s_d, K, I, "row", rank, world)

        def all_reduce(Y):
            dist.all_reduce(Y, op=dist.ReduceOp.SUM)

        GU_r = _oracle_linear(X, (p_gu, s_gu, 2 * (b - a)))
        Y = parallel.tp_mlp(X, (p_gu, s_gu, 2 * (b - a)), (p_dr, s_dr, K), _oracle_linear,
                            _mlp_oracle_act_linear, all_reduce, rank, world)
        out_q.put((rank, (GU_r.numpy(), Y.numpy())))
    finally:
        dist.destroy_process_group()


def test_tp_mlp_gloo_fused_silu_quant():
    """TP FFN (world 2): each rank's [gate_r | up_r] equals the 1-GPU gate / up outputs on its rows (bit
    for bit: column-parallel), SiLU·mul + quantization stays rank-local on that pair, and the all-reduced
    down output matches the fp64 sum of the per-rank exact partials within tolerance."""
    M, I, K, world = 4, 256, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mlp_worker, args=(r, world, port, M, I, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Wg, Wu, Wd = _mlp_weights(I, K)
    X = synth.activations_fp16(M, K, seed=7)
    gate = _oracle_linear(X, (*oracle.quantize_weights(Wg), I)).numpy()
    up = _oracle_linear(X, (*oracle.quantize_weights(Wu), I)).numpy()
    ref = np.zeros((M, K))
    for r in range(world):
        a, b = parallel.gate_up_shard_rows(I, r, world)
        GU_r = res[r][0]
        assert np.array_equal(GU_r[:, : b - a].view(np.uint16), gate[:, a:b].view(np.uint16))
        assert np.array_equal(GU_r[:, b - a:].view(np.uint16), up[:, a:b].view(np.uint16))
        p_d, s_d = oracle.quantize_weights(Wd)
        p_dr, s_dr = parallel.shard_packed(p_d, s_d, K, I, "row", r, world)
        qx, sx, _ = oracle.silu_mul_quantize(np.ascontiguousarray(GU_r))
        ref += oracle.epilogue_f64(oracle.acc_from_packed(qx, p_dr, K, I // world), sx, s_dr)
    assert np.array_equal(res[0][1].view(np.uint16), res[1][1].view(np.uint16))   # all ranks agree
    y = res[0][1].astype(np.float64)
    assert np.all(np.abs(y - ref) <= RTOL * np.abs(ref) + ATOL)


# ---- the benchmark step's own TP path (parallel.rank_layer_plan / shard_layer / tp_decode_layer: the
# functions bench.py runs on GPUs) over gloo, world 2, with the oracle as the rank-local linear ----

TINY = [("qkv", 512, 256, "col"), ("o", 256, 256, "row"), ("gate", 512, 256, "col"), ("up", 512, 256, "col"),
        ("down", 256, 512, "row")]


def _step_inputs(M):
    shapes = synth.fuse_gate_up(TINY)
    Ks = {parallel.QUANT_GROUP[n]: K for n, N, K, kind in shapes}
    return shapes, {qg: synth.activations_fp16(M, K, seed=11 + K) for qg, K in Ks.items()}


def _step_weights(shapes):
    """Full weights, quantized once (oracle packer); gate_up is the fused [gate; up] weight."""
    out = []
    for i, (name, N, K, kind) in enumerate(shapes):
        W = synth.weights_fp16(N, K, seed=40 + i, std_scale=0.25)
        out.append(oracle.quantize_weights(W))
    return out


def _step_linear(X_r, shard, entry):
    name, Nr, Kr, N, K, kind, qg = entry
    p, s0 = shard
    return _oracle_linear(np.ascontiguousarray(X_r), (np.ascontiguousarray(p), np.ascontiguousarray(s0), Nr))


def _step_worker(rank, world, port, M, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shapes, inputs = _step_inputs(M)
        plan = parallel.rank_layer_plan(shapes, world)
        shards = parallel.shard_layer(_step_weights(shapes), plan, rank, world)

        def all_reduce(Y):
            dist.all_reduce(Y, op=dist.ReduceOp.SUM)

        out = parallel.tp_decode_layer(inputs, shards, plan, _step_linear, all_reduce, rank, world)
        out_q.put((rank, {k: v.numpy() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


def test_bench_step_tp_path_gloo():
    """bench.py's decode layer at TP = 2 (gloo, oracle per rank): qkv / gate_up column shards are
    bit-identical to the 1-GPU result on their rows ([gate_r | up_r] for the fused gate_up), o / down are
    all-reduced fp16 partials within tolerance of the fp64 sum of the per-rank exact results, every rank
    ends with the same reduced outputs, and TP = 1 through the same function reproduces the 1-GPU layer."""
    M, world = 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shapes, inputs = _step_inputs(M)
    full = _step_weights(shapes)
    plan1 = parallel.rank_layer_plan(shapes, 1)
    one = {k: v.numpy() for k, v in parallel.tp_decode_layer(inputs, parallel.shard_layer(full, plan1, 0, 1), plan1,
                                                            _step_linear, None, 0, 1).items()}
    # column-parallel: bit-identical slices
    a0 = one["qkv"].shape[1] // 2
    assert np.array_equal(np.concatenate([res[0]["qkv"], res[1]["qkv"]], 1).view(np.uint16), one["qkv"].view(np.uint16))
    I = one["gate_up"].shape[1] // 2
    for r in range(world):
        a, b = parallel.gate_up_shard_rows(I, r, world)
        gu = res[r]["gate_up"]
        assert np.array_equal(gu[:, : b - a].view(np.uint16), one["gate_up"][:, a:b].view(np.uint16))
        assert np.array_equal(gu[:, b - a:].view(np.uint16), one["gate_up"][:, I + a:I + b].view(np.uint16))
    # row-parallel: all ranks agree; within tolerance of the exact per-rank sum; close to 1 GPU
    plan2 = parallel.rank_layer_plan(shapes, world)
    for name in ("o", "down"):
        assert np.array_equal(res[0][name].view(np.uint16), res[1][name].view(np.uint16))
        i = [e[0] for e in plan2].index(name)
        ref = 0
        for r in range(world):
            p_r, s0_r = parallel.shard_layer(full, plan2, r, world)[i]
            X_r = np.ascontiguousarray(parallel.shard_input(inputs[plan2[i][6]], "row", r, world))
            ref = ref + oracle.linear_rows(X_r, p_r, s0_r, plan2[i][1])
        y = res[0][name].astype(np.float64)
        assert np.all(np.abs(y - ref) <= RTOL * np.abs(ref) + ATOL), name
        assert np.linalg.norm(y - one[name]) / np.linalg.norm(one[name]) < 0.05
    assert a0 > 0


def _fused_step_worker(rank, world, port, M, out_q):
    """bench.py's fused-reduction step (NEXT-3) with the oracle as the rank's device: a row-parallel linear
    returns the REDUCED output itself (its partial, gathered from every rank, summed in rank order as
    qoq_w4a8_gemm_allreduce does), so tp_decode_layer(fused_rows=True) issues no separate all-reduce."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shapes, inputs = _step_inputs(M)
        plan = parallel.rank_layer_plan(shapes, world)
        shards = parallel.shard_layer(_step_weights(shapes), plan, rank, world)

        def linear(X_r, shard, entry):
            Y = _step_linear(X_r, shard, entry)
            if entry[5] != "row":
                return Y
            parts = [torch.empty_like(Y) for _ in range(world)]
            dist.all_gather(parts, Y)
            return torch.from_numpy(oracle.tp_reduce_rank_order([p.numpy() for p in parts]))

        def no_collective(Y):
            raise AssertionError("fused_rows must not issue a separate all-reduce")

        out = parallel.tp_decode_layer(inputs, shards, plan, linear, no_collective, rank, world, fused_rows=True)
        out_q.put((rank, {k: v.numpy() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


def test_fused_reduction_step_gloo():
    """The NEXT-3 step at TP = 2: every rank ends with bit-identical o / down outputs (rank-order fp32 sum of
    the fp16 partials, reading Q32), within tolerance of the fp64 sum of the per-rank exact results."""
    M, world = 8, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_step_worker, args=(r, world, port, M, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shapes, inputs = _step_inputs(M)
    full = _step_weights(shapes)
    plan = parallel.rank_layer_plan(shapes, world)
    for name in ("o", "down"):
        assert np.array_equal(res[0][name].view(np.uint16), res[1][name].view(np.uint16))
        i = [e[0] for e in plan].index(name)
        _, Nr, Kr, N, K, kind, qg = plan[i]
        refs = []
        for r in range(world):
            p_r, s0_r = parallel.shard_layer(full, plan, r, world)[i]
            X_r = np.ascontiguousarray(parallel.shard_input(inputs[qg], kind, r, world))
            qx, sx, tx = oracle.quantize_activations(X_r)
            refs.append(oracle.epilogue_f64(oracle.acc_from_packed(qx, np.ascontiguousarray(p_r), N, Kr), sx,
                                            np.ascontiguousarray(s0_r)))
        ref = sum(refs)
        y = res[0][name].astype(np.float64)
        # each fp16 partial within the north_star tolerance of its exact value, plus the final fp16 rounding
        bound = sum(RTOL * np.abs(r) + ATOL for r in refs) + 2.0 ** -11 * np.abs(ref)
        assert np.all(np.abs(y - ref) <= bound)

