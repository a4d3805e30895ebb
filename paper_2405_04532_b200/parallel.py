"""Megatron-style tensor parallelism for the W4A8 linear layers (north_star).

  * column-parallel (qkv, gate/up): W split along N (output channels). Each rank holds rows
    [r N/TP, (r+1) N/TP), quantizes the replicated X exactly as 1 GPU would, and produces its
    N-slice of Y. No collective. The slice is bit-identical to the 1-GPU result (reading Q17).
  * row-parallel (o, down): W split along K (input channels) at 128-group boundaries. Each rank's
    input X_r is the K-shard of X (already sharded by the previous layer); it is quantized with a
    per-rank per-token scale, the rank emits an fp16 partial Y_r = fp16(acc_r s_x^r s0), and the
    partials are summed with ONE all-reduce over the TP group (NCCL over NVLink/NVSwitch on GPUs).

Only sharding / reduction plumbing lives here; every arithmetic step of the path runs in the CUDA
library (paper_2405_04532_b200). Functions that compute take the per-rank `linear` callable, so the
same host logic is exercised by the gloo tests on CPU (tests/test_tp_gloo.py) and by bench.py on GPUs.
"""
from __future__ import annotations

GROUP = 128


def check_shardable(N: int, K: int, kind: str, world: int) -> None:
    if kind == "col":
        if N % (GROUP * world):
            raise ValueError(f"column-parallel N={N} not divisible into {world} shards of 128-multiples")
    elif kind == "row":
        if K % (GROUP * world):
            raise ValueError(f"row-parallel K={K} not divisible into {world} shards at group boundaries")
    else:
        raise ValueError(kind)


def shard_bounds(total: int, rank: int, world: int) -> tuple[int, int]:
    step = total // world
    return rank * step, (rank + 1) * step


def shard_weight(W, kind: str, rank: int, world: int):
    """The rank's shard of an nn.Linear weight W[N][K] (any 2-D array/tensor supporting slicing)."""
    N, K = W.shape
    check_shardable(N, K, kind, world)
    if kind == "col":
        a, b = shard_bounds(N, rank, world)
        return W[a:b]
    a, b = shard_bounds(K, rank, world)
    return W[:, a:b]


TILE_BYTES = 8448


def shard_packed(packed, s0, N: int, K: int, kind: str, rank: int, world: int):
    """Shard an already-packed weight (quantize once, offline, then distribute). The tile stream is
    [N/128][K/128][8448] (include/qoq_b200.h): a column shard is the contiguous block of its 128-row
    tiles (+ its rows of s0); a row shard gathers, for every row block, the k-tiles of its K range
    (s0 stays the full per-channel vector: level 1 is per output channel over ALL of K)."""
    check_shardable(N, K, kind, world)
    NT, KT = N // GROUP, K // GROUP
    tiles = packed.reshape(NT, KT, TILE_BYTES)
    if kind == "col":
        a, b = shard_bounds(NT, rank, world)
        return tiles[a:b].reshape(-1), s0[a * GROUP:b * GROUP]
    a, b = shard_bounds(KT, rank, world)
    sub = tiles[:, a:b]
    sub = sub.contiguous() if hasattr(sub, "contiguous") else sub.copy()
    return sub.reshape(-1), s0


def shard_input(X, kind: str, rank: int, world: int):
    """Column-parallel layers see the replicated X; row-parallel layers see the K-shard of X."""
    if kind == "col":
        return X
    K = X.shape[1]
    a, b = shard_bounds(K, rank, world)
    return X[:, a:b]


def tp_linear(X, W_shard, kind: str, linear, all_reduce, rank: int, world: int):
    """One TP linear layer on this rank.

    linear(X_r, W_shard) -> Y_r  (the rank-local W4A8 linear: quantize X_r per token + GEMM)
    all_reduce(Y) -> in-place SUM over the TP group (row-parallel only)
    Returns the rank's N-slice (col) or the full, reduced Y (row)."""
    X_r = shard_input(X, kind, rank, world)
    Y = linear(X_r, W_shard)
    if kind == "row" and world > 1:
        all_reduce(Y)
    return Y


def gate_up_shard_rows(I: int, rank: int, world: int) -> tuple[int, int]:
    """Rows of gate (and of up) a rank holds in the fused column-parallel gate_up weight [2I][K]: its
    shard is [gate[a:b]; up[a:b]], so its output is [gate_r | up_r] and SiLU(gate)·up stays rank-local."""
    if I % (GROUP * world):
        raise ValueError(f"intermediate size {I} not divisible into {world} shards of 128-multiples")
    return shard_bounds(I, rank, world)


def tp_mlp(X, gate_up_shard, down_shard, linear, act_linear, all_reduce, rank: int, world: int):
    """The TP FFN of Fig. 7 on this rank: column-parallel gate_up (no collective), SiLU(gate)·up on the
    rank's [gate_r | up_r] with the per-token quantization fused in (NEXT-2; per-rank scales over the
    I-shard, reading Q17), row-parallel down, ONE all-reduce.

    linear(X, W_shard) -> fp16 Y (quantize X per token + W4A8 GEMM)
    act_linear(GU_r, W_shard) -> fp16 partial of down (silu_mul_quantize of GU_r + W4A8 GEMM)"""
    GU_r = linear(X, gate_up_shard)
    Y = act_linear(GU_r, down_shard)
    if world > 1:
        all_reduce(Y)
    return Y


# ------------------------------------------------------------------ the decode step's layer under TP
# (one code path for bench.py on GPUs and tests/test_tp_gloo.py on CPU)

QUANT_GROUP = {"qkv": "attn_in", "o": "attn_out", "gate": "mlp_in", "up": "mlp_in", "gate_up": "mlp_in",
               "down": "mlp_act"}


def rank_layer_plan(shapes, world: int):
    """Per-rank GEMMs of one layer: [(name, N_r, K_r, N, K, kind, quant_group)] for the model's
    [(name, N, K, kind)] (gate and up possibly fused into gate_up). Column-parallel layers split N,
    row-parallel layers split K, both at 128 boundaries; quant_group names the activation quantization
    that feeds the GEMM (gate and up share one, Fig. 7)."""
    out = []
    for name, N, K, kind in shapes:
        check_shardable(N // 2 if name == "gate_up" else N, K, kind, world)
        Nr, Kr = (N // world, K) if kind == "col" else (N, K // world)
        out.append((name, Nr, Kr, N, K, kind, QUANT_GROUP[name]))
    return out


def shard_packed_gate_up(packed, s0, I: int, K: int, rank: int, world: int):
    """The rank's shard of a fused, packed [gate; up] weight (N = 2I): the tiles of gate rows [a, b) then
    those of up rows [a, b) (gate_up_shard_rows), so the rank's output is [gate_r | up_r]."""
    a, b = gate_up_shard_rows(I, rank, world)
    NT, KT = 2 * I // GROUP, K // GROUP
    tiles = packed.reshape(NT, KT, TILE_BYTES)
    ga, gb, ua, ub = a // GROUP, b // GROUP, (I + a) // GROUP, (I + b) // GROUP
    if hasattr(tiles, "contiguous"):      # torch
        import torch
        p = torch.cat([tiles[ga:gb], tiles[ua:ub]]).reshape(-1)
        s = torch.cat([s0[a:b], s0[I + a:I + b]])
    else:                                 # numpy
        import numpy as np
        p = np.concatenate([tiles[ga:gb], tiles[ua:ub]]).reshape(-1)
        s = np.concatenate([s0[a:b], s0[I + a:I + b]])
    return p, s


def shard_layer(packed_layer, plan, rank: int, world: int):
    """Per-rank shards [(packed_r, s0_r)] of one layer's full packed weights [(packed, s0)] (quantize once
    on the full weight, then distribute: the same quantized weights as 1 GPU)."""
    out = []
    for (packed, s0), (name, Nr, Kr, N, K, kind, qg) in zip(packed_layer, plan):
        if world == 1:
            out.append((packed, s0))
        elif name == "gate_up" and kind == "col":
            out.append(shard_packed_gate_up(packed, s0, N // 2, K, rank, world))
        else:
            out.append(shard_packed(packed, s0, N, K, kind, rank, world))
    return out


def tp_decode_layer(inputs, shards, plan, linear, all_reduce, rank: int, world: int, fused_rows: bool = False):
    """One decode layer of the benchmark step on this rank, in order (qkv, o, gate_up, down):
    X = inputs[quant_group] (replicated [M][K]; a row-parallel rank reads its K-shard view), then
    Y = linear(X_r, shard, plan_entry) (quantize X_r per token + W4A8 GEMM), then one all_reduce of Y after
    each row-parallel linear — unless fused_rows: then the row-parallel `linear` already returns the reduced
    Y (qoq_w4a8_gemm_allreduce, NEXT-3) and no separate collective runs. Returns {name: Y}."""
    out = {}
    for shard, entry in zip(shards, plan):
        name, Nr, Kr, N, K, kind, qg = entry
        X_r = shard_input(inputs[qg], kind, rank, world)
        Y = linear(X_r, shard, entry)
        if kind == "row" and world > 1 and not fused_rows:
            all_reduce(Y)
        out[name] = Y
    return out


# ------------------------------------------------------------------ fused TP reduction (NEXT-3)

def fused_tp_comm(qoq, group, m_cap: int, n_cap: int, device):
    """The rank's qoq.TpComm over `group`: one symmetric-memory receive buffer per rank (torch.distributed's
    _symmetric_memory: peer-mapped over NVLink), zeroed, exchanged with a rendezvous, so every rank's buffer
    is addressable from every GPU. Collective over `group`."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    nbytes = qoq.tp_recv_bytes(world, m_cap, n_cap)
    if nbytes <= 0:
        raise ValueError("unsupported fused-reduction capacity")
    buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
    buf.zero_()
    hdl = symm_mem.rendezvous(buf, group)
    torch.cuda.synchronize(device)
    dist.barrier(group)          # every rank's buffer is zero before any peer pushes into it
    return qoq.TpComm(rank, world, [int(p) for p in hdl.buffer_ptrs], m_cap, n_cap, device, keep=(buf, hdl))
