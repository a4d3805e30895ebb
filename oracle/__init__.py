"""CPU oracle for the QoQ W4A8 hot path (QServe, arXiv 2405.04532) — numpy front-end over the
plain-C library in qoq_oracle.c.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package. It shares no code with the product path
(paper_2405_04532_b200/, include/) and never imports it. Functions cite the paper passage they
follow (P:n = PAPER.md line n); every function is pinned by tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qoq_oracle.c")
_HDR = os.path.join(_HERE, "qoq_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

TILE_BYTES = 8448
PC_TILE_BYTES = 8192


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no fast-math; OpenMP over GEMM outputs)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-fopenmp", "-shared",
                               "-fPIC", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.c_void_p
            I = ctypes.c_int
            sig = {
                "oracle_h2f": (ctypes.c_float, [ctypes.c_uint16]),
                "oracle_f2h_rn": (ctypes.c_uint16, [ctypes.c_float]),
                "oracle_rhai": (I, [I, I]),
                "oracle_level1": (I, [P, I, I, P, P]),
                "oracle_level2_group": (I, [P, I, P, P, P]),
                "oracle_level2": (I, [P, I, I, I, P, P, P]),
                "oracle_dequant_level2": (I, [P, P, P, I, I, I, P]),
                "oracle_pack": (I, [P, P, P, I, I, I, P]),
                "oracle_unpack": (I, [P, I, I, I, P, P, P]),
                "oracle_quantize_activations": (I, [P, I, I, I, P, P, P]),
                "oracle_gemm_i32": (I, [P, P, I, I, I, I, I, P]),
                "oracle_epilogue_f64": (I, [P, P, P, I, I, P]),
                "oracle_linear_rows": (I, [P, I, I, I, I, P, P, I, P]),
                "oracle_num_threads": (I, []),
                "oracle_set_num_threads": (None, [I]),
                "oracle_pc_quantize": (I, [P, I, I, P, P, P]),
                "oracle_pc_pack": (I, [P, I, I, P]),
                "oracle_pc_unpack": (I, [P, I, I, P]),
                "oracle_pc_gemm_i32": (I, [P, P, P, I, I, I, P]),
                "oracle_d2h_rn": (ctypes.c_uint16, [ctypes.c_double]),
                "oracle_rmsnorm_rinv": (ctypes.c_double, [P, I, ctypes.c_double]),
                "oracle_rmsnorm_fp16": (I, [P, I, I, I, P, ctypes.c_double, P]),
                "oracle_rmsnorm_quantize": (I, [P, I, I, I, P, ctypes.c_double, P, P, P]),
                "oracle_silu_f64": (ctypes.c_double, [ctypes.c_double]),
                "oracle_silu_mul_fp16": (I, [P, P, I, I, I, P]),
                "oracle_silu_mul_quantize": (I, [P, P, I, I, I, P, P, P]),
                "oracle_kv4_quantize": (I, [P, I, I, P, P, P]),
                "oracle_kv4_page_bytes": (ctypes.c_size_t, [I, I, I]),
                "oracle_kv4_store": (I, [P, P, P, P, P, P, I, I, I, I, P, P]),
                "oracle_kv4_dequant": (I, [P, P, P, I, I, P]),
                "oracle_attention_f64": (I, [P, P, P, I, I, I, I, P]),
            }
            for name, (res, args) in sig.items():
                f = getattr(L, name)
                f.restype, f.argtypes = res, args
            _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def _u16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    if a.dtype == np.float16:
        return a.view(np.uint16)
    assert a.dtype == np.uint16
    return a


# ---- scalar helpers ----

def h2f(bits: int) -> float:
    return lib().oracle_h2f(int(bits))


def f2h_rn(x: float) -> int:
    return lib().oracle_f2h_rn(float(np.float32(x)))


def rhai(a: int, b: int) -> int:
    return lib().oracle_rhai(int(a), int(b))


# ---- O1..O6 ----

def level1(W: np.ndarray):
    """O1: -> (q8 int8 [N][K], s0 fp16 [N])."""
    W = _u16(W)
    N, K = W.shape
    q8 = np.empty((N, K), np.int8)
    s0 = np.empty(N, np.uint16)
    _check(lib().oracle_level1(_p(W), N, K, _p(q8), _p(s0)), "level1")
    return q8, s0.view(np.float16)


def level2_group(q8: np.ndarray):
    """O2 on one group: -> (qu4 uint8 [g], s_u8 int, z int)."""
    q8 = np.ascontiguousarray(q8, dtype=np.int8)
    qu4 = np.empty(q8.size, np.uint8)
    s = np.zeros(1, np.uint8)
    z = np.zeros(1, np.uint8)
    _check(lib().oracle_level2_group(_p(q8), q8.size, _p(qu4), _p(s), _p(z)), "level2_group")
    return qu4, int(s[0]), int(z[0])


def level2(q8: np.ndarray, g: int = 128):
    """O2 over [N][K]: -> (qu4 [N][K], s_u8 [N][K/g], z [N][K/g])."""
    q8 = np.ascontiguousarray(q8, dtype=np.int8)
    N, K = q8.shape
    qu4 = np.empty((N, K), np.uint8)
    s = np.empty((N, K // g), np.uint8)
    z = np.empty((N, K // g), np.uint8)
    _check(lib().oracle_level2(_p(q8), N, K, g, _p(qu4), _p(s), _p(z)), "level2")
    return qu4, s, z


def dequant_level2(qu4, s_u8, z, g: int = 128) -> np.ndarray:
    """q̂ = (q_u4 - z) * s_u8 (Eq. P:247): int16 [N][K] so overflow past INT8 is visible."""
    qu4 = np.ascontiguousarray(qu4, np.uint8)
    s_u8 = np.ascontiguousarray(s_u8, np.uint8)
    z = np.ascontiguousarray(z, np.uint8)
    N, K = qu4.shape
    qhat = np.empty((N, K), np.int16)
    _check(lib().oracle_dequant_level2(_p(qu4), _p(s_u8), _p(z), N, K, g, _p(qhat)), "dequant")
    return qhat


def pack(qu4, s_u8, z, g: int = 128) -> np.ndarray:
    """O3: tile stream, (N/128)*(K/128)*8448 bytes."""
    qu4 = np.ascontiguousarray(qu4, np.uint8)
    s_u8 = np.ascontiguousarray(s_u8, np.uint8)
    z = np.ascontiguousarray(z, np.uint8)
    N, K = qu4.shape
    out = np.empty((N // 128) * (K // 128) * TILE_BYTES if N % 128 == 0 and K % 128 == 0 else 1,
                   np.uint8)
    _check(lib().oracle_pack(_p(qu4), _p(s_u8), _p(z), N, K, g, _p(out)), "pack")
    return out


def unpack(packed: np.ndarray, N: int, K: int, g: int = 128):
    packed = np.ascontiguousarray(packed, np.uint8)
    qu4 = np.empty((N, K), np.uint8)
    s = np.empty((N, K // g), np.uint8)
    z = np.empty((N, K // g), np.uint8)
    _check(lib().oracle_unpack(_p(packed), N, K, g, _p(qu4), _p(s), _p(z)), "unpack")
    return qu4, s, z


def quantize_weights(W: np.ndarray, g: int = 128):
    """O1 -> O2 -> O3: the offline packer. -> (packed uint8, s0 fp16 [N])."""
    q8, s0 = level1(W)
    qu4, s, z = level2(q8, g)
    return pack(qu4, s, z, g), s0


def quantize_activations(X: np.ndarray, K: int | None = None):
    """O4: -> (qx int8 [M][K], sx fp16 [M], tx int32 [M])."""
    X = _u16(X)
    M, ldx = X.shape
    K = ldx if K is None else K
    qx = np.empty((M, K), np.int8)
    sx = np.empty(M, np.uint16)
    tx = np.empty(M, np.int32)
    _check(lib().oracle_quantize_activations(_p(X), M, K, ldx, _p(qx), _p(sx), _p(tx)),
           "quantize_activations")
    return qx, sx.view(np.float16), tx


def gemm_i32(qx: np.ndarray, qhat: np.ndarray) -> np.ndarray:
    """O5: exact int32 acc [M][N] (raises if a sum leaves int32)."""
    qx = np.ascontiguousarray(qx, np.int8)
    qhat = np.ascontiguousarray(qhat, np.int16)
    M, K = qx.shape
    N = qhat.shape[0]
    acc = np.empty((M, N), np.int32)
    _check(lib().oracle_gemm_i32(_p(qx), _p(qhat), M, N, K, 0, M, _p(acc)), "gemm_i32")
    return acc


def epilogue_f64(acc: np.ndarray, sx: np.ndarray, s0: np.ndarray) -> np.ndarray:
    """O6: y = acc * s_x[m] * s0[n] in fp64 (exact)."""
    acc = np.ascontiguousarray(acc, np.int32)
    M, N = acc.shape
    y = np.empty((M, N), np.float64)
    _check(lib().oracle_epilogue_f64(_p(acc), _p(_u16(sx)), _p(_u16(s0)), M, N, _p(y)), "epilogue")
    return y


def acc_from_packed(qx: np.ndarray, packed: np.ndarray, N: int, K: int) -> np.ndarray:
    """INT32 accumulators of the W4A8 GEMM on already-quantized activations."""
    qu4, s, z = unpack(packed, N, K)
    return gemm_i32(qx, dequant_level2(qu4, s, z))


def linear_rows(X: np.ndarray, packed: np.ndarray, s0: np.ndarray, N: int,
                m0: int = 0, m1: int | None = None, K: int | None = None) -> np.ndarray:
    """Whole layer y_ref[m0:m1] (fp64) from fp16 X and packed weights: O4 -> O3^-1 -> O5 -> O6."""
    X = _u16(X)
    M, ldx = X.shape
    K = ldx if K is None else K
    m1 = M if m1 is None else m1
    y = np.empty((m1 - m0, N), np.float64)
    _check(lib().oracle_linear_rows(_p(X), K, ldx, m0, m1, _p(np.ascontiguousarray(packed)),
                                    _p(_u16(s0)), N, _p(y)), "linear_rows")
    return y


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


# ---- NEXT-1: per-channel W4A8 (§5.2.2) ----

def pc_quantize(W: np.ndarray):
    """PC1 (Eq. 2, per-channel P:134, FP16 scale P:447): -> (qu4 [N][K], s_w fp16 [N], z_w uint8 [N])."""
    W = _u16(W)
    N, K = W.shape
    qu4 = np.empty((N, K), np.uint8)
    s = np.empty(N, np.uint16)
    z = np.empty(N, np.uint8)
    _check(lib().oracle_pc_quantize(_p(W), N, K, _p(qu4), _p(s), _p(z)), "pc_quantize")
    return qu4, s.view(np.float16), z


def pc_pack(qu4: np.ndarray) -> np.ndarray:
    """The O3 nibble stream without level-2 bytes: (N/128)*(K/128)*8192 bytes."""
    qu4 = np.ascontiguousarray(qu4, np.uint8)
    N, K = qu4.shape
    out = np.empty(max(1, (N // 128) * (K // 128) * PC_TILE_BYTES), np.uint8)
    _check(lib().oracle_pc_pack(_p(qu4), N, K, _p(out)), "pc_pack")
    return out


def pc_unpack(packed: np.ndarray, N: int, K: int) -> np.ndarray:
    packed = np.ascontiguousarray(packed, np.uint8)
    qu4 = np.empty((N, K), np.uint8)
    _check(lib().oracle_pc_unpack(_p(packed), N, K, _p(qu4)), "pc_unpack")
    return qu4


def pc_quantize_weights(W: np.ndarray):
    """PC1 -> pack: the per-channel offline packer. -> (packed uint8, s_w fp16 [N], z_w uint8 [N])."""
    qu4, s, z = pc_quantize(W)
    return pc_pack(qu4), s, z


def pc_gemm_i32(qx: np.ndarray, qu4: np.ndarray, z_w: np.ndarray) -> np.ndarray:
    """Eq. (per_channel_qmm) P:454 in integers: acc = sum_k qx (qu4 - z_w) (exact int32)."""
    qx = np.ascontiguousarray(qx, np.int8)
    qu4 = np.ascontiguousarray(qu4, np.uint8)
    z_w = np.ascontiguousarray(z_w, np.uint8)
    M, K = qx.shape
    N = qu4.shape[0]
    acc = np.empty((M, N), np.int32)
    _check(lib().oracle_pc_gemm_i32(_p(qx), _p(qu4), _p(z_w), M, N, K, _p(acc)), "pc_gemm_i32")
    return acc


def pc_acc_from_packed(qx: np.ndarray, packed: np.ndarray, z_w: np.ndarray, N: int, K: int) -> np.ndarray:
    return pc_gemm_i32(qx, pc_unpack(packed, N, K), z_w)


# ---- NEXT-2: activation quantization fused into RMSNorm / SiLU·mul (Fig. 7; Q23-Q26) ----

def d2h_rn(x: float) -> int:
    """binary64 -> binary16 bits, one round-to-nearest-even (Q24)."""
    return lib().oracle_d2h_rn(float(x))


def rmsnorm_rinv(x: np.ndarray, eps: float) -> float:
    """r = 1/sqrt(S/K + eps), S = exact Σx² rounded once to fp64 (Q25). x: one fp16 row."""
    x = _u16(x)
    return lib().oracle_rmsnorm_rinv(_p(x), x.shape[-1], float(eps))


def rmsnorm_fp16(X: np.ndarray, gamma: np.ndarray, eps: float, K: int | None = None) -> np.ndarray:
    """Llama RMSNorm output in fp16: fp16_rn((x·r)·γ) (Q23-Q25). X [M][ldx] -> [M][K]."""
    X, gamma = _u16(X), _u16(gamma)
    M, ldx = X.shape
    K = ldx if K is None else K
    Y = np.empty((M, K), np.uint16)
    _check(lib().oracle_rmsnorm_fp16(_p(X), M, K, ldx, _p(gamma), float(eps), _p(Y)), "rmsnorm_fp16")
    return Y.view(np.float16)


def rmsnorm_quantize(X: np.ndarray, gamma: np.ndarray, eps: float, K: int | None = None):
    """O4 of rmsnorm_fp16 (the fused layernorm + quantization of P:410) -> (qx, sx, tx)."""
    X, gamma = _u16(X), _u16(gamma)
    M, ldx = X.shape
    K = ldx if K is None else K
    qx = np.empty((M, K), np.int8)
    sx = np.empty(M, np.uint16)
    tx = np.empty(M, np.int32)
    _check(lib().oracle_rmsnorm_quantize(_p(X), M, K, ldx, _p(gamma), float(eps), _p(qx), _p(sx), _p(tx)),
           "rmsnorm_quantize")
    return qx, sx.view(np.float16), tx


def silu_f64(g: float) -> float:
    """silu(g) = g / (1 + exp(-g)) in fp64 (Q26)."""
    return lib().oracle_silu_f64(float(g))


def _gate_up(G: np.ndarray, U: np.ndarray | None, K: int | None):
    """(G, U) as two [M][K] arrays, or G = the [M][2K] gate_up output (gate | up) with U None."""
    G = _u16(G)
    if U is None:
        M, ld = G.shape
        K = ld // 2 if K is None else K
        return G, G[:, K:].copy(), M, K
    U = _u16(U)
    M = G.shape[0]
    K = G.shape[1] if K is None else K
    return np.ascontiguousarray(G[:, :K]), np.ascontiguousarray(U[:, :K]), M, K


def silu_mul_fp16(G: np.ndarray, U: np.ndarray | None = None, K: int | None = None) -> np.ndarray:
    """fp16_rn(silu(g)·u) (Q24, Q26) -> [M][K] fp16."""
    G, U, M, K = _gate_up(G, U, K)
    G = np.ascontiguousarray(G[:, :K])
    H = np.empty((M, K), np.uint16)
    _check(lib().oracle_silu_mul_fp16(_p(G), _p(U), M, K, K, _p(H)), "silu_mul_fp16")
    return H.view(np.float16)


def silu_mul_quantize(G: np.ndarray, U: np.ndarray | None = None, K: int | None = None):
    """O4 of silu_mul_fp16 (the fused activation + quantization of P:410) -> (qx, sx, tx)."""
    G, U, M, K = _gate_up(G, U, K)
    G = np.ascontiguousarray(G[:, :K])
    qx = np.empty((M, K), np.int8)
    sx = np.empty(M, np.uint16)
    tx = np.empty(M, np.int32)
    _check(lib().oracle_silu_mul_quantize(_p(G), _p(U), M, K, K, _p(qx), _p(sx), _p(tx)),
           "silu_mul_quantize")
    return qx, sx.view(np.float16), tx


# ---- NEXT-4: KV4 cache + decode attention (§5.3; Q27-Q29) ----

def kv4_quantize(X: np.ndarray):
    """Rows of D fp16 values -> (q u8 [rows][D], s fp16 [rows], z fp16 [rows]) (Q27)."""
    X = _u16(X)
    rows, D = X.shape
    q = np.empty((rows, D), np.uint8)
    s = np.empty(rows, np.uint16)
    z = np.empty(rows, np.uint16)
    _check(lib().oracle_kv4_quantize(_p(X), rows, D, _p(q), _p(s), _p(z)), "kv4_quantize")
    return q, s.view(np.float16), z.view(np.float16)


def kv4_page_bytes(H_kv: int, D: int, P: int) -> int:
    return lib().oracle_kv4_page_bytes(H_kv, D, P)


def kv4_store(k, v, block_table: np.ndarray, n_pages: int, P: int, pages: np.ndarray | None = None):
    """k, v: (q [T][H_kv][D], s [T][H_kv], z [T][H_kv]) -> pages u8 [n_pages * page_bytes] (Q28)."""
    qk, sk, zk = k
    qv, sv, zv = v
    T, H_kv, D = qk.shape
    if pages is None:
        pages = np.zeros(n_pages * kv4_page_bytes(H_kv, D, P), np.uint8)
    bt = np.ascontiguousarray(block_table, np.int32)
    _check(lib().oracle_kv4_store(_p(np.ascontiguousarray(qk)), _p(_u16(sk)), _p(_u16(zk)),
                                  _p(np.ascontiguousarray(qv)), _p(_u16(sv)), _p(_u16(zv)),
                                  T, H_kv, D, P, _p(bt), _p(pages)), "kv4_store")
    return pages


def kv4_dequant(q: np.ndarray, s: np.ndarray, z: np.ndarray) -> np.ndarray:
    shp = q.shape
    q2 = np.ascontiguousarray(q.reshape(-1, shp[-1]))
    out = np.empty(q2.shape, np.float64)
    _check(lib().oracle_kv4_dequant(_p(q2), _p(_u16(s.reshape(-1))), _p(_u16(z.reshape(-1))), q2.shape[0],
                                    q2.shape[1], _p(out)), "kv4_dequant")
    return out.reshape(shp)


def attention_f64(Q: np.ndarray, Khat: np.ndarray, Vhat: np.ndarray) -> np.ndarray:
    """Q [H][D] fp16, Khat/Vhat [T][H_kv][D] fp64 -> O [H][D] fp64 (Q29)."""
    Q = _u16(Q)
    H, D = Q.shape
    T, H_kv, _ = Khat.shape
    O = np.empty((H, D), np.float64)
    _check(lib().oracle_attention_f64(_p(Q), _p(np.ascontiguousarray(Khat, np.float64)),
                                      _p(np.ascontiguousarray(Vhat, np.float64)), T, H, H_kv, D, _p(O)),
           "attention_f64")
    return O


def tp_reduce_rank_order(partials) -> np.ndarray:
    """Row-parallel TP reduction (north_star: "o_proj/down are row-sharded over K, finished by an ... allreduce
    of the FP16 partials"; reading Q17 for the per-rank partial, Q32 for the order): the fp16 partials Y_0 ..
    Y_{R-1} of the ranks, widened to fp32 and summed in RANK ORDER, one IEEE fp32 addition at a time, then
    rounded once to fp16 (RNE). The paper is single-GPU; the order is this build's reading."""
    acc = None
    for y in partials:
        f = np.asarray(y, dtype=np.float16).astype(np.float32)
        acc = f.copy() if acc is None else (acc + f).astype(np.float32)
    return acc.astype(np.float16)
