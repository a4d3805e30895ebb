"""C-ABI library: loads, exports every symbol include/qoq_b200.h declares, and validates arguments
on the host (no compute calls — these run without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "qoq_b200.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qoq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2405_04532_b200 import build
    build.build()
    import paper_2405_04532_b200 as qoq
    return qoq.load()


def test_header_declares_the_paper_calls():
    fns = declared_functions()
    for f in ("qoq_quantize_weights", "qoq_quantize_activations_per_token", "qoq_w4a8_gemm"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib._name]).decode()
    exported = set(re.findall(r"\bT (qoq_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["cuobjdump", "--list-elf", lib._name]).decode()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_103" not in out


def test_status_strings_and_version(lib):
    assert lib.qoq_abi_version() == 7
    for s in range(0, 8):
        assert lib.qoq_status_string(s)


def test_sizes(lib):
    assert lib.qoq_packed_weight_bytes(256, 256, 128) == 4 * 8448
    assert lib.qoq_packed_weight_bytes(4096, 14336, 128) == 30_277_632
    assert lib.qoq_packed_weight_bytes(100, 256, 128) == 0
    assert lib.qoq_packed_weight_bytes(256, 256, 64) == 0
    assert lib.qoq_gemm_workspace_bytes(16, 64, 256) == 0                     # N not a multiple of 128
    assert lib.qoq_linear_host_scratch_bytes(16, 256, 256) >= 16 * 256 * 5
    # fused linear workspace: 256 B sync + q_x + s_x + t_x (+ split-K partials), 256-B aligned parts
    assert lib.qoq_linear_workspace_bytes(16, 256, 256) >= 256 + 16 * 256 + 2 * 256
    assert lib.qoq_linear_workspace_bytes(16, 256, 200) == 0
    assert lib.qoq_linear_workspace_bytes(64, 4096, 4096) % 256 == 0


def test_host_validation_before_any_device_work(lib):
    P = ctypes.c_void_p
    fake = P(1 << 20)
    # group != 128 -> UNSUPPORTED; N % 128 -> SHAPE; ldx < K -> INVALID_ARG (all host-side)
    assert lib.qoq_quantize_weights(fake, 256, 256, 64, fake, 0, fake, None) == 3
    assert lib.qoq_quantize_weights(fake, 200, 256, 128, fake, 0, fake, None) == 2
    assert lib.qoq_quantize_activations_per_token(fake, 4, 256, 128, fake, fake, None, None) == 1
    assert lib.qoq_w4a8_gemm(fake, fake, None, fake, fake, 4, 256, 200, 128, fake, 256, None, 0, None) == 2
    assert lib.qoq_w4a8_gemm(fake, fake, None, fake, fake, 4, 256, 256, 64, fake, 256, None, 0, None) == 3
    assert lib.qoq_w4a8_gemm(fake, fake, None, fake, fake, 4, 256, 256, 128, fake, 100, None, 0, None) == 1
    assert lib.qoq_w4a8_gemm(fake, fake, None, fake, fake, 4, 256, 131072, 128, fake, 256, None, 0, None) == 2
    # fused linear: shape / group / ldx / ldy / alignment / workspace size, all before device work
    Z = ctypes.c_size_t
    big = Z(1 << 30)
    assert lib.qoq_w4a8_linear(fake, 200, 4, 256, 200, 128, fake, fake, fake, 256, fake, big, None) == 2
    assert lib.qoq_w4a8_linear(fake, 256, 4, 256, 256, 64, fake, fake, fake, 256, fake, big, None) == 3
    assert lib.qoq_w4a8_linear(fake, 128, 4, 256, 256, 128, fake, fake, fake, 256, fake, big, None) == 1
    assert lib.qoq_w4a8_linear(fake, 256, 4, 256, 256, 128, fake, fake, fake, 100, fake, big, None) == 1
    assert lib.qoq_w4a8_linear(P((1 << 20) + 8), 256, 4, 256, 256, 128, fake, fake, fake, 256, fake, big,
                               None) == 1                                      # X not 16-B aligned
    assert lib.qoq_w4a8_linear(fake, 256, 4, 256, 256, 128, fake, fake, fake, 256, P((1 << 20) + 16), big,
                               None) == 1                                      # workspace not 256-B aligned
    assert lib.qoq_w4a8_linear(fake, 256, 4, 256, 256, 128, fake, fake, fake, 256, fake, Z(64), None) == 5
    assert lib.qoq_w4a8_linear(fake, 256, 0, 256, 256, 128, fake, fake, fake, 256, fake, Z(0), None) == 0
    # M == 0 is a no-op that never touches the device
    assert lib.qoq_w4a8_gemm(fake, fake, None, fake, fake, 0, 256, 256, 128, fake, 256, None, 0, None) == 0
    assert lib.qoq_quantize_activations_per_token(fake, 0, 256, 256, fake, fake, None, None) == 0


def test_per_channel_sizes_and_validation(lib):
    """Per-channel W4A8 (NEXT-1): 8192-byte tiles; t_x and 4-byte-aligned z_w are required; shape
    errors as the g128 calls — all host-side, before any device work."""
    P = ctypes.c_void_p
    fake = P(1 << 20)
    assert lib.qoq_pc_packed_weight_bytes(256, 256) == 4 * 8192
    assert lib.qoq_pc_packed_weight_bytes(4096, 14336) == 32 * 112 * 8192
    assert lib.qoq_pc_packed_weight_bytes(100, 256) == 0
    assert lib.qoq_pc_quantize_weights(fake, 200, 256, fake, 1 << 20, fake, fake, None) == 2
    assert lib.qoq_pc_quantize_weights(fake, 256, 256, fake, 10, fake, fake, None) == 5
    args = (fake, fake, None, fake, fake, fake, 4, 256, 256, fake, 256, None, 0, None)
    assert lib.qoq_pc_w4a8_gemm(*args) == 1                                  # t_x missing
    assert lib.qoq_pc_w4a8_gemm(fake, fake, fake, fake, fake, P((1 << 20) + 1), 4, 256, 256, fake, 256,
                                None, 0, None) == 1                          # z_w misaligned
    assert lib.qoq_pc_w4a8_gemm(fake, fake, fake, fake, fake, fake, 4, 256, 200, fake, 256,
                                None, 0, None) == 2                          # K % 128
    assert lib.qoq_pc_w4a8_gemm_i32(fake, None, fake, fake, 4, 256, 256, fake, 256, None, 0, None) == 1
    assert lib.qoq_pc_w4a8_gemm(fake, fake, fake, fake, fake, fake, 0, 256, 256, fake, 256,
                                None, 0, None) == 0                          # M == 0: no-op


def test_fused_quantizer_validation(lib):
    """NEXT-2 entries (qoq_rmsnorm_quantize, qoq_silu_mul_quantize): shape / eps / alignment errors
    and the M == 0 no-op, all host-side, before any device work."""
    P, D = ctypes.c_void_p, ctypes.c_double
    fake = P(1 << 20)
    assert lib.qoq_rmsnorm_quantize(fake, 256, fake, D(1e-5), 4, 204, fake, fake, None, None) == 2   # K % 8
    assert lib.qoq_rmsnorm_quantize(fake, 128, fake, D(1e-5), 4, 256, fake, fake, None, None) == 1   # ldx < K
    assert lib.qoq_rmsnorm_quantize(fake, 256, fake, D(-1.0), 4, 256, fake, fake, None, None) == 1   # eps < 0
    assert lib.qoq_rmsnorm_quantize(fake, 256, fake, D(float("nan")), 4, 256, fake, fake, None, None) == 1
    assert lib.qoq_rmsnorm_quantize(fake, 256, P((1 << 20) + 8), D(1e-5), 4, 256, fake, fake, None, None) == 1
    assert lib.qoq_rmsnorm_quantize(fake, 256, fake, D(1e-5), 0, 256, fake, fake, None, None) == 0
    assert lib.qoq_silu_mul_quantize(fake, fake, 512, 4, 252, fake, fake, None, None) == 2
    assert lib.qoq_silu_mul_quantize(fake, fake, 128, 4, 256, fake, fake, None, None) == 1
    assert lib.qoq_silu_mul_quantize(fake, P((1 << 20) + 2), 512, 4, 256, fake, fake, None, None) == 1
    assert lib.qoq_silu_mul_quantize(fake, None, 512, 4, 256, fake, fake, None, None) == 1
    assert lib.qoq_silu_mul_quantize(fake, fake, 512, 0, 256, fake, fake, None, None) == 0


def test_kv4_validation(lib):
    """NEXT-4 entries: page size query, D / GQA-ratio / shape errors and the B == 0 no-op, host-side."""
    P = ctypes.c_void_p
    fake = P(1 << 20)
    assert lib.qoq_kv4_page_bytes(8, 128, 64) == 8 * 64 * 136
    assert lib.qoq_kv4_page_bytes(8, 64, 64) == 0
    assert lib.qoq_kv4_append(fake, fake, fake, 4, 8, 64, 64, fake, None) == 3            # D != 128
    assert lib.qoq_kv4_append(fake, fake, None, 4, 8, 128, 64, fake, None) == 1           # slots missing
    assert lib.qoq_kv4_append(fake, fake, fake, 0, 8, 128, 64, fake, None) == 0
    assert lib.qoq_kv4_append(fake, fake, fake, 4, 8, 128, 48, fake, None) == 3            # page_size % 32
    assert lib.qoq_kv4_append(fake, fake, fake, 4, 8, 128, 512, fake, None) == 3           # page_size > 256
    args = (fake, fake, fake, fake, 4, 32, 8, 128, 64, 16, fake, None)
    assert lib.qoq_kv4_decode_attention(fake, fake, fake, fake, 4, 30, 8, 128, 64, 16, fake, None) == 2
    assert lib.qoq_kv4_decode_attention(fake, fake, fake, fake, 4, 48, 3, 128, 64, 16, fake, None) == 3
    assert lib.qoq_kv4_decode_attention(fake, fake, fake, fake, 4, 32, 8, 128, 64, 0, fake, None) == 1
    assert lib.qoq_kv4_decode_attention(P((1 << 20) + 8), *args[1:]) == 1
    assert lib.qoq_kv4_decode_attention(fake, fake, fake, fake, 0, 32, 8, 128, 64, 16, fake, None) == 0


def test_linear_chain_validation(lib):
    """qoq_w4a8_linear_chain / qoq_linear_chain_workspace_bytes (ABI v6): host-side validation of the
    descriptor array, M and n ranges and the workspace size — all before any device call."""
    import paper_2405_04532_b200 as qoq
    P, Z = ctypes.c_void_p, ctypes.c_size_t
    lib.qoq_linear_chain_workspace_bytes.restype = Z
    lib.qoq_linear_chain_workspace_bytes.argtypes = [ctypes.c_int, ctypes.c_int, P]
    lib.qoq_w4a8_linear_chain.restype = ctypes.c_int
    lib.qoq_w4a8_linear_chain.argtypes = [ctypes.c_int, ctypes.c_int, P, P, Z, P]
    fake = 1 << 20
    D = qoq.LinearDesc
    good = (D * 2)(D(fake, 4096, 6144, 4096, fake, fake, fake, 6144), D(fake, 6144, 4096, 6144, fake, fake, fake, 4096))
    nb = lib.qoq_linear_chain_workspace_bytes(64, 2, good)
    # counters + 2 x split-K partial tiles [NT max = 48][BN = 64][128] i32 + 2 x q_x [KT max = 48][64][128]
    assert nb >= 2 * 48 * 64 * 128 * 4 + 2 * 48 * 64 * 128
    assert lib.qoq_linear_chain_workspace_bytes(0, 2, good) == 0        # M out of range
    assert lib.qoq_linear_chain_workspace_bytes(129, 2, good) == 0
    assert lib.qoq_linear_chain_workspace_bytes(64, 0, good) == 0       # n out of range
    assert lib.qoq_w4a8_linear_chain(64, 2, good, None, Z(nb), None) == 1            # no workspace
    assert lib.qoq_w4a8_linear_chain(64, 2, good, P(fake), Z(nb - 256), None) == 5   # too small
    assert lib.qoq_w4a8_linear_chain(64, 129, good, P(fake), Z(nb), None) == 1       # n > 128
    big_k = (D * 1)(D(fake, 16384, 128, 16384, fake, fake, fake, 128))          # K > 14336 (quantizer staging)
    assert lib.qoq_w4a8_linear_chain(64, 1, big_k, P(fake), Z(1 << 30), None) == 2
    bad_ldy = (D * 1)(D(fake, 4096, 128, 4096, fake, fake, fake, 132))         # ldy % 8 != 0
    assert lib.qoq_w4a8_linear_chain(64, 1, bad_ldy, P(fake), Z(1 << 30), None) == 1
    bad_shape = (D * 1)(D(fake, 4096, 100, 4096, fake, fake, fake, 128))
    assert lib.qoq_w4a8_linear_chain(64, 1, bad_shape, P(fake), Z(1 << 30), None) == 2
    bad_ld = (D * 1)(D(fake, 4000, 128, 4096, fake, fake, fake, 128))            # ldx < K
    assert lib.qoq_w4a8_linear_chain(64, 1, bad_ld, P(fake), Z(1 << 30), None) == 1
    bad_al = (D * 1)(D(fake + 8, 4096, 128, 4096, fake, fake, fake, 128))        # X misaligned
    assert lib.qoq_w4a8_linear_chain(64, 1, bad_al, P(fake), Z(1 << 30), None) == 1
    null_y = (D * 1)(D(fake, 4096, 128, 4096, fake, fake, None, 128))
    assert lib.qoq_w4a8_linear_chain(64, 1, null_y, P(fake), Z(1 << 30), None) == 1


def test_fused_tp_reduction_sizes_and_validation(lib):
    """NEXT-3 entry: capacity query, and every comm / capacity violation rejected on the host."""
    import paper_2405_04532_b200 as qoq
    assert lib.qoq_tp_recv_bytes(8, 64, 4096) == 2 * 8 * 64 * 4096 * 4   # flag-in-data words: 4 B per fp16
    assert lib.qoq_tp_recv_bytes(9, 64, 4096) == 0 and lib.qoq_tp_recv_bytes(2, 64, 100) == 0
    assert lib.qoq_tp_recv_bytes(2, 0, 4096) == 0
    P = ctypes.c_void_p
    fake = P(1 << 20)

    def comm(rank=0, world=2, m_cap=64, n_cap=4096, null=False):
        recv = (ctypes.c_void_p * 8)(*([1 << 20] * 8))
        if null:
            recv[1] = None
        return qoq._TpCommC(recv, 1 << 20, 1 << 20, 1 << 20, rank, world, m_cap, n_cap)

    def call(c, M=64, N=4096, K=512, group=128, ldy=4096):
        return lib.qoq_w4a8_gemm_allreduce(fake, fake, None, fake, fake, M, N, K, group, fake, ldy,
                                           ctypes.byref(c) if c is not None else None, None)

    assert call(None) == 1
    assert call(comm(world=9)) == 1 and call(comm(rank=2)) == 1 and call(comm(rank=-1)) == 1
    assert call(comm(null=True)) == 1
    assert call(comm(m_cap=32)) == 1 and call(comm(n_cap=2048)) == 1 and call(comm(n_cap=4160)) == 1
    assert call(comm(), ldy=4000) == 1
    assert call(comm(), group=64) == 3 and call(comm(), K=500) == 2
    assert call(comm(), M=0) == 0   # nothing to do
