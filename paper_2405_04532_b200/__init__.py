"""B200-native (sm_100a) QoQ W4A8 hot path of QServe (arXiv 2405.04532) — Python binding.

Thin ctypes marshalling over the C ABI in include/qoq_b200.h (libqoq_b200.so, built in-tree):
every step of the path runs in the library's CUDA kernels. PyTorch is used only for device memory,
streams and process groups. There is no CPU fallback: if the library or an sm_100 GPU is missing,
every call raises.

Function names follow the ABI: quantize_weights, quantize_activations_per_token, w4a8_gemm,
w4a8_gemm_i32, linear_host. Tensors are torch tensors on the current CUDA device; calls are
asynchronous on torch's current stream (or `stream=`).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# QOQ_LIB_VARIANT selects a debug/ablation build (tools only); production uses libqoq_b200.so
LIB_PATH = os.path.join(_HERE, "libqoq_b200.so" if not os.environ.get("QOQ_LIB_VARIANT")
                        else f"libqoq_b200_{os.environ['QOQ_LIB_VARIANT']}.so")
GROUP = 128
TILE_BYTES = 8448
ABI_VERSION = 7
# kernels launched per call (matches include/qoq_b200.h)
LAUNCHES = {"quantize_weights": 2, "quantize_activations_per_token": 1, "w4a8_gemm": 1,
            "w4a8_gemm_i32": 1, "pc_quantize_weights": 2, "pc_w4a8_gemm": 1, "pc_w4a8_gemm_i32": 1,
            "rmsnorm_quantize": 1, "silu_mul_quantize": 1, "kv4_append": 1, "kv4_decode_attention": 1,
            "w4a8_linear_chain": 1}
FUSE_MAX_M = 64   # w4a8_linear / linear_host with QOQ_LINEAR_FUSED=1: one fused kernel up to this M


def linear_fused(M: int) -> bool:
    """True when w4a8_linear runs the one-kernel fused path (opt-in: QOQ_LINEAR_FUSED=1, M <= 64)."""
    return M <= FUSE_MAX_M and os.environ.get("QOQ_LINEAR_FUSED") == "1"


def linear_launches(M: int) -> int:
    """Kernels one w4a8_linear (or linear_host) call launches."""
    return 1 if linear_fused(M) else 2

_lock = threading.Lock()
_lib = None


class QoQError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn}: status {status} ({msg})")
        self.status = status


def load() -> ctypes.CDLL:
    """Load libqoq_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        _sync_knobs(_lib)
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        sig = {
            "qoq_status_string": (ctypes.c_char_p, [I]),
            "qoq_abi_version": (I, []),
            "qoq_packed_weight_bytes": (Z, [I, I, I]),
            "qoq_quantize_weights": (I, [P, I, I, I, P, Z, P, P]),
            "qoq_quantize_activations_per_token": (I, [P, I, I, I, P, P, P, P]),
            "qoq_gemm_workspace_bytes": (Z, [I, I, I]),
            "qoq_w4a8_gemm": (I, [P, P, P, P, P, I, I, I, I, P, I, P, Z, P]),
            "qoq_w4a8_gemm_i32": (I, [P, P, P, I, I, I, I, P, I, P, Z, P]),
            "qoq_linear_workspace_bytes": (Z, [I, I, I]),
            "qoq_w4a8_linear": (I, [P, I, I, I, I, I, P, P, P, I, P, Z, P]),
            "qoq_linear_host_scratch_bytes": (Z, [I, I, I]),
            "qoq_linear_host": (I, [P, I, I, P, P, I, P, P, Z, P]),
            "qoq_pc_packed_weight_bytes": (Z, [I, I]),
            "qoq_pc_quantize_weights": (I, [P, I, I, P, Z, P, P, P]),
            "qoq_pc_w4a8_gemm": (I, [P, P, P, P, P, P, I, I, I, P, I, P, Z, P]),
            "qoq_pc_w4a8_gemm_i32": (I, [P, P, P, P, I, I, I, P, I, P, Z, P]),
            "qoq_rmsnorm_quantize": (I, [P, I, P, ctypes.c_double, I, I, P, P, P, P]),
            "qoq_silu_mul_quantize": (I, [P, P, I, I, I, P, P, P, P]),
            "qoq_kv4_page_bytes": (Z, [I, I, I]),
            "qoq_kv4_append": (I, [P, P, P, I, I, I, I, P, P]),
            "qoq_kv4_decode_attention": (I, [P, P, P, P, I, I, I, I, I, I, P, P]),
            "qoq_linear_chain_workspace_bytes": (Z, [I, I, P]),
            "qoq_w4a8_linear_chain": (I, [I, I, P, P, Z, P]),
            "qoq_debug_reload_knobs": (None, []),
            "qoq_tp_recv_bytes": (Z, [I, I, I]),
            "qoq_w4a8_gemm_allreduce": (I, [P, P, P, P, P, I, I, I, I, P, I, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        if L.qoq_abi_version() != ABI_VERSION:
            raise ImportError("libqoq_b200.so ABI version mismatch; rebuild")
        _sync_knobs(L)
        _lib = L
    return _lib


_KNOB_VARS = ("QOQ_FORCE_MODE", "QOQ_BN_BIG", "QOQ_FORCE_CG", "QOQ_LINEAR_FUSED", "QOQ_CHAIN_SMAX", "QOQ_FQ_THREADS")
_knob_seen = None


def _sync_knobs(L):
    """The library reads its QOQ_* test / tuning overrides once; re-read them when they changed here
    (before any size query or launch, so both see the same plan)."""
    global _knob_seen
    cur = tuple(os.environ.get(k) for k in _KNOB_VARS)
    if cur != _knob_seen:
        L.qoq_debug_reload_knobs()
        _knob_seen = cur


def _check(fn: str, rc: int):
    if rc != 0:
        raise QoQError(fn, rc, load().qoq_status_string(rc).decode())


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


# ------------------------------------------------------------------ sizes

def packed_weight_bytes(N: int, K: int, group: int = GROUP) -> int:
    return load().qoq_packed_weight_bytes(N, K, group)


def gemm_workspace_bytes(M: int, N: int, K: int) -> int:
    return load().qoq_gemm_workspace_bytes(M, N, K)


def linear_workspace_bytes(M: int, N: int, K: int) -> int:
    return load().qoq_linear_workspace_bytes(M, N, K)


def linear_workspace_views(ws: torch.Tensor, M: int, N: int, K: int):
    """(qx [M][K] int8, sx [M] fp16, tx [M] int32) views of a qoq_w4a8_linear workspace (header layout:
    [256 B sync][GEMM workspace][q_x][s_x][t_x], each part 256-B aligned)."""
    def up(v):
        return (v + 255) // 256 * 256
    o_qx = 256 + up(gemm_workspace_bytes(M, N, K))
    o_sx = o_qx + up(M * K)
    o_tx = o_sx + up(2 * M)
    qx = ws[o_qx:o_qx + M * K].view(torch.int8).view(M, K)
    sx = ws[o_sx:o_sx + 2 * M].view(torch.float16)
    tx = ws[o_tx:o_tx + 4 * M].view(torch.int32)
    return qx, sx, tx


def linear_host_scratch_bytes(M: int, N: int, K: int) -> int:
    return load().qoq_linear_host_scratch_bytes(M, N, K)


# ------------------------------------------------------------------ the three calls + debug

def quantize_weights(W: torch.Tensor, group: int = GROUP, stream=None):
    """W [N][K] fp16 (cuda) -> (packed uint8 tile stream, s0 fp16 [N])."""
    if W.dtype != torch.float16 or W.dim() != 2:
        raise ValueError("W must be a 2-D fp16 tensor")
    N, K = W.shape
    nbytes = packed_weight_bytes(N, K, group)
    packed = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=W.device)
    s0 = torch.empty(N, dtype=torch.float16, device=W.device)
    _check("qoq_quantize_weights",
           load().qoq_quantize_weights(_ptr(W), N, K, group, _ptr(packed), nbytes, _ptr(s0), _stream(stream)))
    return packed[:nbytes], s0


def quantize_activations_per_token(X: torch.Tensor, K: int | None = None, want_tx: bool = True,
                                   out=None, stream=None):
    """X [M][ldx] fp16 -> (qx int8 [M][K], sx fp16 [M], tx int32 [M] or None)."""
    if X.dtype != torch.float16 or X.dim() != 2:
        raise ValueError("X must be a 2-D fp16 tensor")
    if X.stride(1) != 1 or not X.is_cuda:
        raise ValueError("X must be a CUDA tensor with contiguous rows")
    M = X.shape[0]
    ldx = X.stride(0) if M > 1 else X.shape[1]     # a row-strided view (e.g. a TP K-shard) is fine
    K = X.shape[1] if K is None else K
    if out is None:
        qx = torch.empty(M, K, dtype=torch.int8, device=X.device)
        sx = torch.empty(M, dtype=torch.float16, device=X.device)
        tx = torch.empty(M, dtype=torch.int32, device=X.device) if want_tx else None
    else:
        qx, sx, tx = out
    _check("qoq_quantize_activations_per_token",
           load().qoq_quantize_activations_per_token(ctypes.c_void_p(X.data_ptr()), M, K, ldx, _ptr(qx), _ptr(sx),
                                                     _ptr(tx), _stream(stream)))
    return qx, sx, tx


def _act_out(M: int, K: int, device, want_tx: bool, out):
    if out is not None:
        return out
    return (torch.empty(M, K, dtype=torch.int8, device=device),
            torch.empty(M, dtype=torch.float16, device=device),
            torch.empty(M, dtype=torch.int32, device=device) if want_tx else None)


def rmsnorm_quantize(X: torch.Tensor, gamma: torch.Tensor, eps: float = 1e-5, K: int | None = None,
                     want_tx: bool = True, out=None, stream=None):
    """RMSNorm with the per-token INT8 quantization fused in (NEXT-2; C-ABI
    qoq_rmsnorm_quantize): X [M][ldx] fp16, gamma [K] fp16 -> (qx int8 [M][K], sx fp16 [M], tx)."""
    if X.dtype != torch.float16 or X.dim() != 2 or gamma.dtype != torch.float16:
        raise ValueError("X must be a 2-D fp16 tensor and gamma fp16")
    M, ldx = X.shape
    K = ldx if K is None else K
    qx, sx, tx = _act_out(M, K, X.device, want_tx, out)
    _check("qoq_rmsnorm_quantize",
           load().qoq_rmsnorm_quantize(_ptr(X), ldx, _ptr(gamma), float(eps), M, K, _ptr(qx), _ptr(sx),
                                       _ptr(tx), _stream(stream)))
    return qx, sx, tx


def silu_mul_quantize(gate_up: torch.Tensor, K: int | None = None, want_tx: bool = True, out=None,
                      stream=None):
    """SiLU(gate)·up with the per-token INT8 quantization fused in (NEXT-2; C-ABI
    qoq_silu_mul_quantize). gate_up [M][2K] fp16 is the fused gate_up GEMM output (gate | up)."""
    if gate_up.dtype != torch.float16 or gate_up.dim() != 2:
        raise ValueError("gate_up must be a 2-D fp16 tensor")
    M, ld = gate_up.shape
    K = ld // 2 if K is None else K
    if not gate_up.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    qx, sx, tx = _act_out(M, K, gate_up.device, want_tx, out)
    base = gate_up.data_ptr()
    _check("qoq_silu_mul_quantize",
           load().qoq_silu_mul_quantize(ctypes.c_void_p(base), ctypes.c_void_p(base + 2 * K), ld, M, K,
                                        _ptr(qx), _ptr(sx), _ptr(tx), _stream(stream)))
    return qx, sx, tx


def kv4_page_bytes(H_kv: int, D: int = 128, page_size: int = 64) -> int:
    return load().qoq_kv4_page_bytes(H_kv, D, page_size)


def kv4_append(K: torch.Tensor, V: torch.Tensor, slots: torch.Tensor, pages: torch.Tensor, page_size: int = 64,
               stream=None):
    """Quantize one new token per sequence into the KV4 page pool (NEXT-4; C-ABI qoq_kv4_append).
    K, V [B][H_kv][D] fp16; slots [B] int32 (page * page_size + offset); pages uint8 pool."""
    if K.dim() != 3 or K.shape != V.shape or K.dtype != torch.float16 or V.dtype != torch.float16:
        raise ValueError("K and V must be [B][H_kv][D] fp16 tensors of the same shape")
    B, H_kv, D = K.shape
    if slots.dtype != torch.int32 or slots.numel() != B:
        raise ValueError("slots must be int32 [B]")
    if pages.dtype != torch.uint8:
        raise ValueError("pages must be a uint8 tensor")
    _check("qoq_kv4_append", load().qoq_kv4_append(_ptr(K), _ptr(V), _ptr(slots), B, H_kv, D, page_size,
                                                   _ptr(pages), _stream(stream)))


def kv4_decode_attention(Q: torch.Tensor, pages: torch.Tensor, block_table: torch.Tensor, seq_lens: torch.Tensor,
                         H_kv: int, page_size: int = 64, out=None, stream=None):
    """Decode attention over the KV4 cache (§5.3; C-ABI qoq_kv4_decode_attention): Q [B][H][D] fp16 ->
    O [B][H][D] fp16."""
    if Q.dim() != 3 or Q.dtype != torch.float16:
        raise ValueError("Q must be a [B][H][D] fp16 tensor")
    B, H, D = Q.shape
    if pages.dtype != torch.uint8:
        raise ValueError("pages must be a uint8 tensor")
    if block_table.dtype != torch.int32 or block_table.dim() != 2 or block_table.shape[0] != B:
        raise ValueError("block_table must be int32 [B][max_pages]")
    if seq_lens.dtype != torch.int32 or seq_lens.numel() != B:
        raise ValueError("seq_lens must be int32 [B]")
    O = torch.empty_like(Q) if out is None else out
    if O.shape != Q.shape or O.dtype != torch.float16:
        raise ValueError("out must be fp16 with Q's shape")
    _check("qoq_kv4_decode_attention",
           load().qoq_kv4_decode_attention(_ptr(Q), _ptr(pages), _ptr(block_table), _ptr(seq_lens), B, H, H_kv,
                                           D, page_size, block_table.shape[1], _ptr(O), _stream(stream)))
    return O


class Workspace:
    """Zero-filled workspace that grows on demand. A GEMM workspace is left zeroed by the library; a
    linear (w4a8_linear) workspace additionally holds the last call's q_x / s_x / t_x, so do not pass
    the same Workspace to both kinds of call, nor to concurrent calls on different streams."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int, stream=None):
        """The buffer (grown and zero-filled on `stream`, the stream the call launches on)."""
        if nbytes == 0:
            return None, 0
        if self.buf is None or self.buf.numel() < nbytes:
            s = torch.cuda.current_stream(self.device) if stream is None else stream
            with torch.cuda.stream(s):
                self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=self.device or "cuda")
        return self.buf, self.buf.numel()


_default_ws: dict = {}


def _ws_for(device, nbytes, workspace, kind="gemm", stream=None):
    """Default workspaces are per (device, LAUNCH stream, kind): calls on different streams never share
    one (a GEMM workspace holds split-K partials and tile counters that must be zero on entry), and it
    is allocated and zero-filled on the stream the kernel runs on. A linear workspace also holds the
    call's quantized activations, so the two kinds never share a buffer."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    if workspace is None:
        key = (str(device), s.cuda_stream, kind)
        workspace = _default_ws.setdefault(key, Workspace(device))
    if isinstance(workspace, Workspace):
        return workspace.get(nbytes, s)
    return workspace.get(nbytes)


def w4a8_gemm(qx: torch.Tensor, sx: torch.Tensor, tx: torch.Tensor | None, packed: torch.Tensor,
              s0: torch.Tensor, N: int, out: torch.Tensor | None = None, workspace: Workspace | None = None,
              stream=None) -> torch.Tensor:
    """Y [M][N] fp16 = fp16(s_x[m] s0[n] Σ_k qx[m][k] q̂[n][k])."""
    M, K = qx.shape
    Y = torch.empty(M, N, dtype=torch.float16, device=qx.device) if out is None else out
    ws, wsb = _ws_for(qx.device, gemm_workspace_bytes(M, N, K), workspace, stream=stream)
    _check("qoq_w4a8_gemm",
           load().qoq_w4a8_gemm(_ptr(qx), _ptr(sx), _ptr(tx), _ptr(packed), _ptr(s0), M, N, K, GROUP,
                                _ptr(Y), Y.stride(0), _ptr(ws), wsb, _stream(stream)))
    return Y


def w4a8_gemm_i32(qx: torch.Tensor, tx: torch.Tensor | None, packed: torch.Tensor, N: int,
                  workspace: Workspace | None = None, stream=None) -> torch.Tensor:
    """Exact INT32 accumulators acc [M][N] (parity/debug entry)."""
    M, K = qx.shape
    acc = torch.empty(M, N, dtype=torch.int32, device=qx.device)
    ws, wsb = _ws_for(qx.device, gemm_workspace_bytes(M, N, K), workspace, stream=stream)
    _check("qoq_w4a8_gemm_i32",
           load().qoq_w4a8_gemm_i32(_ptr(qx), _ptr(tx), _ptr(packed), M, N, K, GROUP, _ptr(acc), N,
                                    _ptr(ws), wsb, _stream(stream)))
    return acc


def w4a8_linear(X: torch.Tensor, packed: torch.Tensor, s0: torch.Tensor, N: int, K: int | None = None,
                out: torch.Tensor | None = None, workspace: Workspace | None = None, stream=None) -> torch.Tensor:
    """Y [M][N] fp16 = w4a8_gemm(quantize_activations_per_token(X)) bit for bit; ONE fused kernel for
    M <= 64 (quantization in the GEMM's prologue), quantizer + GEMM above. X [M][ldx] fp16, K <= ldx."""
    if X.dtype != torch.float16 or X.dim() != 2:
        raise ValueError("X must be a 2-D fp16 tensor")
    M, ldx = X.shape
    K = ldx if K is None else K
    Y = torch.empty(M, N, dtype=torch.float16, device=X.device) if out is None else out
    ws, wsb = _ws_for(X.device, linear_workspace_bytes(M, N, K), workspace, kind="linear", stream=stream)
    _check("qoq_w4a8_linear",
           load().qoq_w4a8_linear(_ptr(X), ldx, M, N, K, GROUP, _ptr(packed), _ptr(s0), _ptr(Y), Y.stride(0),
                                  _ptr(ws), wsb, _stream(stream)))
    return Y


def linear(X: torch.Tensor, packed: torch.Tensor, s0: torch.Tensor, N: int, K: int | None = None,
           workspace: Workspace | None = None, stream=None) -> torch.Tensor:
    """The W4A8 linear layer: per-token quantization + GEMM (w4a8_linear)."""
    return w4a8_linear(X, packed, s0, N, K, workspace=workspace, stream=stream)


def linear_host(X_host: torch.Tensor, packed: torch.Tensor, s0: torch.Tensor, N: int,
                Y_host: torch.Tensor, scratch: torch.Tensor, stream=None):
    """End-to-end through the C ABI with pinned HOST X/Y: H2D, w4a8_linear, D2H (async)."""
    if X_host.is_cuda or Y_host.is_cuda:
        raise ValueError("linear_host takes host tensors")
    M, K = X_host.shape
    _check("qoq_linear_host",
           load().qoq_linear_host(ctypes.c_void_p(X_host.data_ptr()), M, K, _ptr(packed), _ptr(s0), N,
                                  ctypes.c_void_p(Y_host.data_ptr()), _ptr(scratch), scratch.numel(),
                                  _stream(stream)))


# ------------------------------------------------------------------ per-channel W4A8 (NEXT-1, §5.2.2)

def pc_packed_weight_bytes(N: int, K: int) -> int:
    return load().qoq_pc_packed_weight_bytes(N, K)


def pc_quantize_weights(W: torch.Tensor, stream=None):
    """W [N][K] fp16 (cuda) -> (packed uint8 8192-byte tiles, s_w fp16 [N], z_w uint8 [N])."""
    if W.dtype != torch.float16 or W.dim() != 2:
        raise ValueError("W must be a 2-D fp16 tensor")
    N, K = W.shape
    nbytes = pc_packed_weight_bytes(N, K)
    packed = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=W.device)
    s_w = torch.empty(N, dtype=torch.float16, device=W.device)
    z_w = torch.empty(max(N, 4), dtype=torch.uint8, device=W.device)
    _check("qoq_pc_quantize_weights",
           load().qoq_pc_quantize_weights(_ptr(W), N, K, _ptr(packed), nbytes, _ptr(s_w), _ptr(z_w),
                                          _stream(stream)))
    return packed[:nbytes], s_w, z_w[:N]


def pc_w4a8_gemm(qx: torch.Tensor, sx: torch.Tensor, tx: torch.Tensor, packed: torch.Tensor, s_w: torch.Tensor,
                 z_w: torch.Tensor, N: int, out: torch.Tensor | None = None, workspace: Workspace | None = None,
                 stream=None) -> torch.Tensor:
    """Y [M][N] fp16 = fp16(s_x[m] s_w[n] (Σ_k qx q_u4 − z_w[n] t_x[m]))."""
    M, K = qx.shape
    Y = torch.empty(M, N, dtype=torch.float16, device=qx.device) if out is None else out
    ws, wsb = _ws_for(qx.device, gemm_workspace_bytes(M, N, K), workspace, stream=stream)
    _check("qoq_pc_w4a8_gemm",
           load().qoq_pc_w4a8_gemm(_ptr(qx), _ptr(sx), _ptr(tx), _ptr(packed), _ptr(s_w), _ptr(z_w), M, N, K,
                                   _ptr(Y), Y.stride(0), _ptr(ws), wsb, _stream(stream)))
    return Y


def pc_w4a8_gemm_i32(qx: torch.Tensor, tx: torch.Tensor, packed: torch.Tensor, z_w: torch.Tensor, N: int,
                     workspace: Workspace | None = None, stream=None) -> torch.Tensor:
    """Exact INT32 Σ_k qx (q_u4 − z_w) [M][N] (parity entry)."""
    M, K = qx.shape
    acc = torch.empty(M, N, dtype=torch.int32, device=qx.device)
    ws, wsb = _ws_for(qx.device, gemm_workspace_bytes(M, N, K), workspace, stream=stream)
    _check("qoq_pc_w4a8_gemm_i32",
           load().qoq_pc_w4a8_gemm_i32(_ptr(qx), _ptr(tx), _ptr(packed), _ptr(z_w), M, N, K, _ptr(acc), N,
                                       _ptr(ws), wsb, _stream(stream)))
    return acc


# ------------------------------------------------------------------ decode chain (one persistent launch)

class LinearDesc(ctypes.Structure):
    """qoq_linear_desc (include/qoq_b200.h)."""
    _fields_ = [("X", ctypes.c_void_p), ("ldx", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
                ("packed", ctypes.c_void_p), ("s0", ctypes.c_void_p), ("Y", ctypes.c_void_p), ("ldy", ctypes.c_int)]


def chain_descs(layers):
    """layers: [(X [M][ldx] fp16, packed, s0, N, Y [M][ldy] fp16, K or None)] -> (M, ctypes array)."""
    M = None
    arr = (LinearDesc * len(layers))()
    for i, L in enumerate(layers):
        X, packed, s0, N, Y = L[:5]
        K = L[5] if len(L) > 5 and L[5] is not None else X.shape[1]
        if X.dtype != torch.float16 or Y.dtype != torch.float16 or X.dim() != 2 or Y.dim() != 2:
            raise ValueError("X and Y must be 2-D fp16 tensors")
        if X.stride(1) != 1 or Y.stride(1) != 1:
            raise ValueError("X and Y rows must be contiguous")
        if M is None:
            M = X.shape[0]
        if X.shape[0] != M or Y.shape[0] != M or Y.shape[1] < N:
            raise ValueError("every linear of a chain takes the same M tokens; Y must be [M][>= N]")
        arr[i] = LinearDesc(X.data_ptr(), X.stride(0), N, K, _ptr(packed).value, _ptr(s0).value, Y.data_ptr(),
                            Y.stride(0))
    return M, arr


def linear_chain_workspace_bytes(layers) -> int:
    M, arr = chain_descs(layers)
    return load().qoq_linear_chain_workspace_bytes(M, len(arr), arr)


def w4a8_linear_chain(layers, workspace: Workspace | None = None, stream=None):
    """Y_j = w4a8_linear(X_j) for every linear j of `layers`, in order, in ONE persistent kernel (C-ABI
    qoq_w4a8_linear_chain; M <= 128). X_j may be an earlier Y_i (read after it is complete).
    layers: [(X, packed, s0, N, Y[, K])]."""
    M, arr = chain_descs(layers)
    nbytes = load().qoq_linear_chain_workspace_bytes(M, len(arr), arr)
    if nbytes == 0:
        raise ValueError("unsupported chain (M must be 1..128, n 1..128, shapes multiples of 128, K <= 14336)")
    dev = layers[0][0].device
    ws, wsb = _ws_for(dev, nbytes, workspace, kind="chain", stream=stream)
    _check("qoq_w4a8_linear_chain", load().qoq_w4a8_linear_chain(M, len(arr), arr, _ptr(ws), wsb, _stream(stream)))


# ------------------------------------------------------------------ fused TP reduction (NEXT-3, ABI v7)

TP_MAX_WORLD = 8


class _TpCommC(ctypes.Structure):
    """include/qoq_b200.h qoq_tp_comm."""
    _fields_ = [("recv", ctypes.c_void_p * 8), ("gen", ctypes.c_void_p), ("done", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("rank", ctypes.c_int), ("world", ctypes.c_int), ("m_cap", ctypes.c_int),
                ("n_cap", ctypes.c_int)]


def tp_recv_bytes(world: int, m_cap: int, n_cap: int) -> int:
    return int(load().qoq_tp_recv_bytes(world, m_cap, n_cap))


class TpComm:
    """One rank's fused TP reduction (qoq_tp_comm): every rank's receive-buffer pointer (as mapped on this GPU)
    and this rank's counters. The receive buffers are allocated and shared by the caller (parallel.fused_tp_comm:
    symmetric memory over the TP group; `local`: one rank)."""

    def __init__(self, rank: int, world: int, recv_ptrs, m_cap: int, n_cap: int, device, keep=()):
        if not 1 <= world <= TP_MAX_WORLD or not 0 <= rank < world:
            raise ValueError("need 0 <= rank < world <= 8")
        self.rank, self.world, self.m_cap, self.n_cap = rank, world, m_cap, n_cap
        ptrs = [int(v) for v in recv_ptrs]
        if len(ptrs) != world:
            raise ValueError("one receive buffer per rank")
        self.ctr = torch.zeros(64, dtype=torch.int32, device=device)   # gen | done | status (64 B apart)
        self._keep = keep
        base = self.ctr.data_ptr()
        self._c = _TpCommC((ctypes.c_void_p * 8)(*ptrs), base, base + 64, base + 128, rank, world, m_cap, n_cap)

    @classmethod
    def local(cls, m_cap: int, n_cap: int, device):
        """world = 1: the reduction of one partial (Y equals w4a8_gemm bit for bit)."""
        recv = torch.zeros(tp_recv_bytes(1, m_cap, n_cap), dtype=torch.uint8, device=device)
        return cls(0, 1, [recv.data_ptr()], m_cap, n_cap, device, keep=(recv,))

    def status(self) -> int:
        """1 if a wait for a peer timed out (after synchronizing)."""
        return int(self.ctr[32].item())

    def calls(self) -> int:
        return int(self.ctr[0].item())


def w4a8_gemm_allreduce(qx: torch.Tensor, sx: torch.Tensor, tx: torch.Tensor | None, packed: torch.Tensor,
                        s0: torch.Tensor, N: int, comm: TpComm, out: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """Row-parallel W4A8 GEMM with the TP reduction fused into its epilogue: Y = fp16(Σ_q fp32(Y_q)) over the
    ranks of `comm`, summed in rank order, identical on every rank (include/qoq_b200.h)."""
    M, K = qx.shape
    Y = torch.empty(M, N, dtype=torch.float16, device=qx.device) if out is None else out
    _check("qoq_w4a8_gemm_allreduce",
           load().qoq_w4a8_gemm_allreduce(_ptr(qx), _ptr(sx), _ptr(tx), _ptr(packed), _ptr(s0), M, N, K, GROUP,
                                          _ptr(Y), Y.stride(0), ctypes.byref(comm._c), _stream(stream)))
    return Y
