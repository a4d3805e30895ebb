"""GPU parity for the KV4 cache and decode attention (NEXT-4, §5.3; readings
Q27-Q29) through the C ABI against the CPU oracle: pages written by qoq_kv4_append BYTE-exact with the
oracle's quantizer + page layout (across page boundaries, permuted block tables); attention within the
per-element tolerance derived from the kernel's fp32 arithmetic (tests/kv4_tol.py: fp16 output
rounding, fp32 score / softmax / accumulation error bounds, per head and channel) of the fp64 attention
over the oracle's dequantized cache, for every GQA ratio, ragged lengths (1, P-1, P, P+1, ...), empty sequences and the
bench configuration (B = 64, 1024 tokens, Llama-3-8B heads)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from kv4_tol import kv4_tolerance

pytestmark = pytest.mark.gpu
D, P = 128, 64


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")


def kv_rows(T, H_kv, seed, scale=1.0):
    x = synth.normal(seed, 5, T * H_kv * D).reshape(T, H_kv, D) * scale
    x[:, :, 3] *= 8.0                                                   # an outlier channel
    return x.astype(np.float16)


def oracle_cache(Ks, Vs, tables, n_pages, P=P):
    """Ks/Vs: per sequence [T][H_kv][D] fp16 -> (pages, [(Khat, Vhat)])."""
    H_kv = Ks[0].shape[1]
    pages = np.zeros(n_pages * oracle.kv4_page_bytes(H_kv, D, P), np.uint8)
    deq = []
    for K, V, bt in zip(Ks, Vs, tables):
        T = K.shape[0]
        if T == 0:
            deq.append(None)
            continue
        k = oracle.kv4_quantize(K.reshape(-1, D))
        v = oracle.kv4_quantize(V.reshape(-1, D))
        shp = lambda a: a.reshape(T, H_kv, *a.shape[1:])
        oracle.kv4_store(tuple(shp(a) for a in k), tuple(shp(a) for a in v), bt, n_pages, P, pages)
        deq.append((oracle.kv4_dequant(*k).reshape(T, H_kv, D), oracle.kv4_dequant(*v).reshape(T, H_kv, D)))
    return pages, deq


def tables_for(lens, seed, P=P):
    need = [max(1, -(-T // P)) for T in lens]
    n_pages = sum(need) + 3
    perm = np.random.default_rng(seed).permutation(n_pages)
    maxp = max(need)
    bt = np.zeros((len(lens), maxp), np.int32)
    o = 0
    for b, n in enumerate(need):
        bt[b, :n] = perm[o:o + n]
        o += n
    return bt, n_pages


@pytest.mark.parametrize("B,H_kv,T", [(3, 8, 70), (2, 1, 129), (4, 2, 1)])
def test_kv4_append_pages_byte_exact(gpu_lib, B, H_kv, T):
    bt, n_pages = tables_for([T] * B, seed=T)
    Ks = [kv_rows(T, H_kv, 10 + b) for b in range(B)]
    Vs = [kv_rows(T, H_kv, 20 + b, scale=0.5) for b in range(B)]
    if T > 2:
        Ks[0][1, 0] = 0.25                                               # constant row: s = 1 rule
        Vs[0][2, 0] = 0                                                  # zero row
    ref, _ = oracle_cache(Ks, Vs, bt, n_pages)
    pages = torch.zeros(n_pages * gpu_lib.kv4_page_bytes(H_kv, D, P), dtype=torch.uint8, device="cuda:0")
    for t in range(T):
        Kt = to_dev(np.stack([K[t] for K in Ks]))
        Vt = to_dev(np.stack([V[t] for V in Vs]))
        slots = to_dev(np.array([bt[b, t // P] * P + t % P for b in range(B)], np.int32))
        gpu_lib.kv4_append(Kt, Vt, slots, pages, P)
    torch.cuda.synchronize()
    got = pages.cpu().numpy()
    bad = np.flatnonzero(got != ref)
    assert bad.size == 0, f"{bad.size} page bytes differ, first at {bad[:8].tolist()}"


def check_attention(gpu_lib, lens, H, H_kv, seed, P=P):
    B = len(lens)
    bt, n_pages = tables_for(lens, seed, P)
    Ks = [kv_rows(T, H_kv, seed + 100 + b) for b, T in enumerate(lens)]
    Vs = [kv_rows(T, H_kv, seed + 200 + b, scale=0.7) for b, T in enumerate(lens)]
    pages, deq = oracle_cache(Ks, Vs, bt, n_pages, P)
    Q = (synth.normal(seed, 6, B * H * D).reshape(B, H, D) * 2.0).astype(np.float16)
    O = gpu_lib.kv4_decode_attention(to_dev(Q), to_dev(pages), to_dev(bt), to_dev(np.array(lens, np.int32)),
                                     H_kv, P)
    torch.cuda.synchronize()
    o = O.cpu().numpy().astype(np.float64)
    for b, T in enumerate(lens):
        if T == 0:
            assert np.all(o[b] == 0)
            continue
        Kh, Vh = deq[b]
        ref = oracle.attention_f64(Q[b], Kh, Vh)
        tol = kv4_tolerance(Q[b], Kh, Vh, ref)
        err = np.abs(o[b] - ref)
        assert np.all(err <= tol), f"seq {b} (T={T}): max err/tol {(err / tol).max()}"


@pytest.mark.parametrize("H,H_kv", [(32, 8), (8, 8), (16, 8), (16, 2)])
def test_kv4_attention_gqa_ratios(gpu_lib, H, H_kv):
    check_attention(gpu_lib, [1, 63, 64, 65, 200], H, H_kv, seed=H * 10 + H_kv)


def test_kv4_attention_ragged_and_empty(gpu_lib):
    check_attention(gpu_lib, [0, 5, 1, 128, 0, 777], 32, 8, seed=3)


def test_kv4_attention_bench_size_sampled(gpu_lib):
    """The bench configuration: B = 64 sequences x 1024 tokens, Llama-3-8B heads (H = 32, H_kv = 8);
    the whole batch runs on the GPU, 6 sequences are checked against the fp64 oracle."""
    B, T, H, H_kv = 64, 1024, 32, 8
    lens = [T] * B
    bt, n_pages = tables_for(lens, 9)
    sample = [0, 1, 17, 31, 50, 63]
    Ks = [kv_rows(T, H_kv, 300 + b) if b in sample else np.zeros((T, H_kv, D), np.float16) for b in range(B)]
    Vs = [kv_rows(T, H_kv, 400 + b, 0.7) if b in sample else np.zeros((T, H_kv, D), np.float16) for b in range(B)]
    pages, deq = oracle_cache(Ks, Vs, bt, n_pages)
    Q = (synth.normal(9, 6, B * H * D).reshape(B, H, D) * 2.0).astype(np.float16)
    O = gpu_lib.kv4_decode_attention(to_dev(Q), to_dev(pages), to_dev(bt), to_dev(np.array(lens, np.int32)), H_kv, P)
    torch.cuda.synchronize()
    o = O.cpu().numpy().astype(np.float64)
    for b in sample:
        Kh, Vh = deq[b]
        ref = oracle.attention_f64(Q[b], Kh, Vh)
        err = np.abs(o[b] - ref)
        assert np.all(err <= kv4_tolerance(Q[b], Kh, Vh, ref)), (b, err.max())


@pytest.mark.parametrize("page", [32, 256])
def test_kv4_attention_page_sizes(gpu_lib, page):
    """Other page sizes: 32 (the smallest allowed) and 256 (the largest: 3 staged pages of 34.8 KB in
    shared memory, past the default 48 KB)."""
    check_attention(gpu_lib, [1, page - 1, page, page + 1, 3 * page + 5], 32, 8, seed=page, P=page)


def test_kv4_attention_peaked_outlier_data(gpu_lib):
    """The smoke test's data: Q, K and V with 4 input channels scaled x20 (synth.activations_fp16), so the
    softmax is sharply peaked and most p·s_V are far below fp16's normal range — the PV operand must keep
    its relative precision there (bf16 terms) for the derived tolerance to hold."""
    T, H, H_kv, P_ = 70, 8, 2, 64
    Kx = synth.activations_fp16(T * H_kv, D, seed=2).reshape(T, H_kv, D)
    Vx = synth.activations_fp16(T * H_kv, D, seed=3).reshape(T, H_kv, D)
    bt = np.array([[1, 0]], np.int32)
    pages, deq = oracle_cache([Kx], [Vx], bt, 2, P_)
    Q = synth.activations_fp16(H, D, seed=4).reshape(1, H, D)
    O = gpu_lib.kv4_decode_attention(to_dev(Q), to_dev(pages), to_dev(bt), to_dev(np.array([T], np.int32)), H_kv, P_)
    torch.cuda.synchronize()
    Kh, Vh = deq[0]
    ref = oracle.attention_f64(Q[0], Kh, Vh)
    err = np.abs(O.cpu().numpy()[0].astype(np.float64) - ref)
    tol = kv4_tolerance(Q[0], Kh, Vh, ref)
    assert np.all(err <= tol), f"max err/tol {(err / tol).max()}"
